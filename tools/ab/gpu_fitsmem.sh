AGR_LIB_PATH=$PWD/build/var/new/libagr.so timeout 900 python -m pytest tests/test_bvh_gpu.py tests/test_parity_gpu.py -m gpu -x -q -k "bvh or update or c6 or fit or mesh" 2>&1 | tail -1
for r in 1 2 3; do for v in old new; do bash tools/runab.sh fit_${v}_$r $v "--config 6 --no-table2 --no-counters"; done; done
