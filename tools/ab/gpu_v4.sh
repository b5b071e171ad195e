AGR_LIB_PATH=$PWD/build/var/new/libagr.so timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for c in 3 4 5; do bash tools/runvar.sh v4_c${c}_$r "--config $c --no-table2" old new; done; done
