AGR_LIB_PATH=$PWD/build/var/r2v/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -2
bash tools/runvar.sh rplc_c3 "--config 3 --no-table2" base r2v r2h r2v13
bash tools/runvar.sh rplc_c4 "--config 4 --no-table2" base r2v r2h
bash tools/runvar.sh rplc_c5 "--config 5 --no-table2" base r2v
bash tools/ab/gpu_rpl2_prof.sh
