timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
bash tools/runvar.sh triv_c6_$r "--config 6 --no-table2" old new
bash tools/runvar.sh triv_c3_$r "--config 3 --no-table2" old new
done
