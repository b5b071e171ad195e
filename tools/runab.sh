#!/bin/bash
# usage: runab.sh tag lib "argsA" "argsB" ... : bench variants on the same box
tag=$1; lib=$2; shift 2
i=0
for a in "$@"; do
  AGR_LIB_PATH=$PWD/build/var/$lib/libagr.so python bench.py --no-cpu-baseline --no-e2e $a > gpurun_out/${tag}_$i.json 2> gpurun_out/${tag}_$i.err
  python - "$a" "gpurun_out/${tag}_$i.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    c=d.get("counters_per_ray") or {}
    print(repr(sys.argv[1]), "%.4g"%d["value"], "cast %.3f upd %.3f"%(d["cast_ms_per_step"], d["update_ms_per_step"]), {k: round(v,3) for k,v in c.items() if k in ("nodes","leaves","instances","tlas_nodes")})
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  i=$((i+1))
done
