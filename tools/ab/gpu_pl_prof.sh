B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 --config 6"
AGR_LIB_PATH=$PWD/build/var/pl16s16/libagr.so timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_cast \
   --launch-skip 3 --launch-count 1 -f -o gpurun_out/pl_c6 $B > gpurun_out/pl_ncu.log 2>&1
tail -2 gpurun_out/pl_ncu.log
