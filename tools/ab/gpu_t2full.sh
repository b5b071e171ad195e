timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "warp_path or refit or tlas_builders or max_instances" 2>&1 | tail -2
timeout 900 python bench.py --table2 > gpurun_out/r02o_table2.json 2> gpurun_out/r02o_table2.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02o_table2.json').read().strip().splitlines()[-1])
rows={}
for c in d["table2"]["cells"]:
    rows.setdefault((c["res"],c["mode"]),{})[c["envs"]]=c["env_frames_per_sec"]
for k,v in rows.items(): print(k, "  ".join("%d:%.3g"%(e,f) for e,f in sorted(v.items())))
PY
