for r in 1 2; do bash tools/runvar.sh occ3_c3_$r "--config 3 --no-table2 --no-counters" b16 b15 b14; bash tools/runvar.sh occ3_c5_$r "--config 5 --no-table2 --no-counters" b16 b15 b14; done
