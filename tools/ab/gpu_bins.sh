for c in 3; do
  echo "== c$c"
  bash tools/runvar.sh bins_c$c "--config $c --no-table2" s48 s64 s48 s64
done
timeout 300 python bench.py --config 3 --no-table2 --no-cpu-baseline --no-e2e --no-counters --steps 3 > /dev/null 2> gpurun_out/bins_err.txt; echo rc $?
