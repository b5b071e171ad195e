timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tw_gputests.txt 2>&1; tail -2 gpurun_out/tw_gputests.txt
for c in 4 5; do timeout 600 python bench.py --config $c --no-table2 --no-cpu-baseline --no-e2e --no-counters > gpurun_out/tw_c$c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/tw_c$c.json').read().strip().splitlines()[-1]); print('c$c', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']))"; done
timeout 600 python bench.py --config 5 --tlas-step refit --no-table2 --no-cpu-baseline --no-e2e --no-counters > gpurun_out/tw_c5r.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/tw_c5r.json').read().strip().splitlines()[-1]); print('c5 refit', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']))"
timeout 600 python bench.py --table2 --t2-res 8x8,64x64 --t2-envs 128,2048 > gpurun_out/tw_t2.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/tw_t2.json').read().strip().splitlines()[-1])
for c in d['table2']['cells']: print(c['res'], c['envs'], c['mode'], '%.4f ms'%c['ms_per_step'])"
