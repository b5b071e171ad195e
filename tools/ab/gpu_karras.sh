timeout 900 python -m pytest tests/test_bvh_gpu.py tests/test_parity_gpu.py -m gpu -x -q -k "karras or bvh or update or c6" 2>&1 | tail -2
for r in 1 2 3; do bash tools/runab.sh kar_old_$r old "--config 6 --no-table2 --no-counters"; bash tools/runab.sh kar_new_$r new "--config 6 --no-table2 --no-counters"; done
