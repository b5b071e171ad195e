for c in 3 4 5; do
  echo "== c$c"
  bash tools/runvar.sh l2_c$c "--config $c --no-table2" base l2p base l2p
done
