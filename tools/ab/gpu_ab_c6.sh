for v in base full; do
  if [ $v = base ]; then L=$PWD/paper_2503_01471_b200/lib/libagr.so; else L=$PWD/build/var/$v/libagr.so; fi
  AGR_LIB_PATH=$L timeout 600 python bench.py --config 6 --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/ab_c6_$v.json 2>&1
  AGR_LIB_PATH=$L timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_c6_$v.csv python bench.py --config 6 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 > /dev/null 2>&1
done
