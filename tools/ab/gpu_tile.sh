for c in 4 3; do
  echo "== c$c"
  bash tools/runvar.sh tile_c$c "--config $c --no-table2" tw4 tw8
done
