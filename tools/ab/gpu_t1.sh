timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "single_and_degenerate or degenerate_faces" 2>&1 | tail -3
