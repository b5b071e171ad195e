timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/dp_gputests.txt 2>&1; tail -2 gpurun_out/dp_gputests.txt
for c in 3 4 5; do
timeout 600 python bench.py --config $c --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/dp_c$c.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/dp_c$c.json').read().strip().splitlines()[-1]); c=d['counters_per_ray']; print('c$c', '%.4g'%d['value'], 'cast %.3f'%d['cast_ms_per_step'], {k: round(c[k],3) for k in ('nodes','leaves','instances','tlas_nodes')})"
done
timeout 600 python bench.py --config 6 --traversal auto --no-table2 --no-cpu-baseline --no-e2e --no-counters > gpurun_out/dp_c6a.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/dp_c6a.json').read().strip().splitlines()[-1]); print('c6 auto', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']))"
