timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "bench_step_full_size" --durations=5 2>&1 | tail -8
