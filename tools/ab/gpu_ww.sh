echo "== c6"; bash tools/runvar.sh ww_c6 "--config 6 --no-table2" w0 w1 w0 w1
for v in w0 w1; do AGR_LIB_PATH=$PWD/build/var/$v/libagr.so timeout 600 python bench.py --table2 --t2-res 8x8,32x32,64x64 --t2-envs 128,2048 > gpurun_out/ww_t2_$v.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ww_t2_$v.json').read().strip().splitlines()[-1]); print('$v', [(c['res'],c['envs'],round(c['ms_per_step_l2_warm']*1e3,1)) for c in d['table2']['cells'] if c['mode']=='static'])"; done
AGR_LIB_PATH=$PWD/build/var/w1/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "c6 or wide or lane or update_mesh or rays_random or edge" 2>&1 | tail -2
