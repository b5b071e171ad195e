for c in 3 4 5; do
  echo "== c$c"
  bash tools/runvar.sh tdp_c$c "--config $c --no-table2" t15 t30 t50
done
