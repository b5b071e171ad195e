AGR_LIB_PATH=$PWD/build/var/pc1/libagr.so timeout 1300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for c in 3 4 5; do bash tools/runvar.sh pc_c${c}_$r "--config $c --no-table2" pc0 pc1; done; done
