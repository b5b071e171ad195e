AGR_LIB_PATH=$PWD/build/var/t2/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "c3 or c5 or wide_tile or bvh8" 2>&1 | tail -1
for r in 1 2; do for c in 3 5; do bash tools/runvar.sh tile3_c${c}_$r "--config $c --no-table2" t4 t2; done; done
