for r in 1 2 3; do bash tools/runvar.sh pc4_$r "--config 4 --no-table2" pc0 new; done
bash tools/runvar.sh pc4_c5 "--config 5 --no-table2" new
