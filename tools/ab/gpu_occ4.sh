for r in 1 2; do
bash tools/runvar.sh occ4_c3_$r "--config 3 --no-table2 --no-counters" b14 b12
bash tools/runvar.sh occ4_c4_$r "--config 4 --no-table2 --no-counters" b16 b14 b12
bash tools/runvar.sh occ4_c6_$r "--config 6 --no-table2 --no-counters" b16 b14
done
