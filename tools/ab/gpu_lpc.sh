AGR_LIB_PATH=$PWD/build/var/lpc1/libagr.so timeout 1300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for v in main lpc1 lpc0; do bash tools/runab.sh lpc_${v}_$r $v "--config 6 --no-table2"; done; done
for v in main lpc1; do bash tools/runab.sh lpc3_$v $v "--config 3 --no-table2 --no-counters"; done
