AGR_LIB_PATH=$PWD/build/var/pair/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "bvh8 or wide or c3 or c5" 2>&1 | tail -2
for r in 1 2; do
for c in 3 4 5; do bash tools/runvar.sh pair_c${c}_$r "--config $c --no-table2" head split pair; done
done
