# ncu capture of the two-rays-per-lane cast (c3) for the source view
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 --config 3"
AGR_LIB_PATH=$PWD/build/var/r2v/libagr.so timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_cast \
   --launch-skip 3 --launch-count 1 -f -o gpurun_out/rpl2_c3 $B > gpurun_out/rpl2_ncu.log 2>&1
tail -3 gpurun_out/rpl2_ncu.log
