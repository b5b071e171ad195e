timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/q_gputests.txt 2>&1; tail -2 gpurun_out/q_gputests.txt
for c in 3 4 5; do
timeout 600 python bench.py --config $c --no-table2 --no-cpu-baseline --no-e2e --no-counters > gpurun_out/q_c$c.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/q_c$c.json').read().strip().splitlines()[-1]); print('c$c', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']), d['clocks'])"
done
