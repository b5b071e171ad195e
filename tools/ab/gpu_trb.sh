for r in 3 6 10; do
timeout 600 python bench.py --config 3 --trbvh-rounds $r --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/trb_$r.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/trb_$r.json').read().strip().splitlines()[-1]); c=d['counters_per_ray']; print('$r', '%.4g'%d['value'], 'cast %.3f'%d['cast_ms_per_step'], {k: round(c[k],3) for k in ('nodes','leaves','instances','tlas_nodes')})"
done
