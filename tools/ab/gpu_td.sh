timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/td_gputests.txt 2>&1; tail -2 gpurun_out/td_gputests.txt
for t in lane auto; do
timeout 600 python bench.py --config 6 --traversal $t --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/td_c6_$t.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/td_c6_$t.json').read().strip().splitlines()[-1]); print('$t', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']))"
done
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/td_launches_c6.csv python bench.py --config 6 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 > /dev/null 2>&1
