AGR_LIB_PATH=$PWD/build/var/pb14/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "lidar or beams or dome or c4" 2>&1 | tail -1
for r in 1 2; do bash tools/runvar.sh beams_$r "--config 4 --no-table2 --no-counters" base pb14 pb16 nb14; done
