for t in lane auto packet4; do
timeout 600 python bench.py --config 6 --traversal $t --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/c6t_$t.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/c6t_$t.json').read().strip().splitlines()[-1]); c=d['counters_per_ray']; print('$t', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']), {k: round(c[k],2) for k in ('nodes','leaves','instances')})"
done
