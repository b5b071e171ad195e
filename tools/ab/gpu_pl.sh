# persistent lanes (k_cast_pl) vs the static per-lane schedule: parity subset, then c6 and the
# Table-II small cameras (per-lane in auto mode)
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "c6 or lane or mode or wide_tile or schedule or update or host" 2>&1 | tail -2
for r in 1 2; do
  bash tools/runab.sh pl_c6_$r pl0 "--config 6 --no-table2"
  for v in pl16 pl8 pl24; do bash tools/runab.sh pl_c6_${v}_$r $v "--config 6 --no-table2"; done
done
for v in pl0 pl16; do
  AGR_LIB_PATH=$PWD/build/var/$v/libagr.so timeout 600 python bench.py --table2 > gpurun_out/pl_t2_$v.json 2>&1
  python - gpurun_out/pl_t2_$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
cells=d.get("table2",d).get("cells",[]) if isinstance(d.get("table2",d),dict) else []
print(sys.argv[2], [(c["res"],c["envs"],c["mode"],round(c["ms_per_step"],4)) for c in cells][:12])
PY
done
