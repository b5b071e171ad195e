timeout 600 python bench.py --config 6 --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/c6x_bench_c6.json 2> gpurun_out/c6x_bench_c6.err
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c6x_launches_c6.csv python bench.py --config 6 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 > /dev/null 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
   -k "regex:k_fit|k_bvh4_topdown|k_pack_tris|k_karras" -c 4 -f -o gpurun_out/c6x_build \
   python bench.py --config 6 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 > gpurun_out/c6x_ncu.log 2>&1
