for c in 3 4 5; do
  echo "== c$c"
  bash tools/runvar.sh rk_c$c "--config $c --no-table2" r0 r1 r2
done
