for r in 1 2; do for c in 4 5; do for w in 8 32; do
  timeout 600 python bench.py --config $c --node-width $w --no-table2 --no-cpu-baseline --no-e2e > gpurun_out/w32c45_c${c}_$w.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/w32c45_c${c}_$w.json').read().strip().splitlines()[-1]); c=d['counters_per_ray']; print('c$c w$w', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']), {k: round(c[k],3) for k in ('nodes','leaves','instances','tlas_nodes')})"
done; done; done
