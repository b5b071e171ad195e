timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --config 6 --no-table2 --no-cpu-baseline --no-e2e --no-counters > gpurun_out/x_c6.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/x_c6.json').read().strip().splitlines()[-1]); print('c6', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']))"
