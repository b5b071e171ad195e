for v in r1 r0 r1 r0; do
  AGR_LIB_PATH=$PWD/build/var/$v/libagr.so timeout 600 python bench.py --config 6 --no-table2 --no-cpu-baseline --no-e2e --no-counters > gpurun_out/rec_$v.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/rec_$v.json').read().strip().splitlines()[-1]); print('$v lane', '%.4g'%d['value'], 'upd %.3f cast %.3f'%(d['update_ms_per_step'], d['cast_ms_per_step']))"
done
AGR_LIB_PATH=$PWD/build/var/r0/libagr.so timeout 900 python -m pytest tests/test_bvh_gpu.py tests/test_parity_gpu.py -m gpu -x -q -k "bvh or update_mesh or c6 or parts or trbvh or degenerate" 2>&1 | tail -2
