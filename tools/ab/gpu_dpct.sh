for c in 3 4; do
  echo "== c$c"
  bash tools/runvar.sh dpct_c$c "--config $c --no-table2" c045 c065 c090 c130
done
