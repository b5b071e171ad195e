mkdir -p build/var/base && cp paper_2503_01471_b200/lib/libagr.so build/var/base/
for c in 3 5; do
  echo "== c$c"
  bash tools/runvar.sh oc2_c$c "--config $c --no-table2" base b18 b20
done
