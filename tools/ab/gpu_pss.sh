AGR_LIB_PATH=$PWD/build/var/pss18/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "bvh8 or wide or c3 or c5" 2>&1 | tail -2
for r in 1 2; do
bash tools/runvar.sh pss_c3_$r "--config 3 --no-table2" base pss16 pss18 pss19 b18
bash tools/runvar.sh pss_c4_$r "--config 4 --no-table2" base pss16 pss18 pss19
done
