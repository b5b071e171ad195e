# GPU tests + c6/c3 bench after BLAS build changes
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c6w_gputests.txt 2>&1
tail -5 gpurun_out/c6w_gputests.txt
timeout 600 python bench.py --config 6 --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/c6w_bench_c6.json 2> gpurun_out/c6w_bench_c6.err
timeout 600 python bench.py --config 3 --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/c6w_bench_c3.json 2> gpurun_out/c6w_bench_c3.err
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c6w_launches_c6.csv python bench.py --config 6 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 > /dev/null 2>&1
tail -2 gpurun_out/c6w_bench_c6.err
