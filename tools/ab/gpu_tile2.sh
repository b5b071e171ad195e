timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 3 4; do
timeout 600 python bench.py --config $c --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/tl_c$c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/tl_c$c.json').read().strip().splitlines()[-1]); c=d['counters_per_ray']; print('c$c', '%.4g'%d['value'], 'cast %.3f'%d['cast_ms_per_step'], {k: round(c[k],3) for k in ('nodes','leaves','instances')})"
done
