timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/b8c_gputests.txt 2>&1; tail -2 gpurun_out/b8c_gputests.txt
for t in lane auto; do
timeout 600 python bench.py --config 6 --traversal $t --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/b8c_c6_$t.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/b8c_c6_$t.json').read().strip().splitlines()[-1]); print('$t', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']))"
done
timeout 600 python bench.py --config 3 --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/b8c_c3.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/b8c_c3.json').read().strip().splitlines()[-1]); c=d['counters_per_ray']; print('c3', '%.4g'%d['value'], 'cast %.3f'%d['cast_ms_per_step'], {k: round(c[k],3) for k in ('nodes','leaves','tlas_nodes')})"
