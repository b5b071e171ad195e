#!/bin/bash
# usage: runvar.sh tag "bench args" v0 v1 ...
tag=$1; args=$2; shift 2
for v in "$@"; do
  AGR_LIB_PATH=$PWD/build/var/$v/libagr.so python bench.py --no-cpu-baseline --no-e2e $args > gpurun_out/${tag}_$v.json 2> gpurun_out/${tag}_$v.err
  python - "$v" "gpurun_out/${tag}_$v.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    c=d.get("counters_per_ray") or {}
    print(sys.argv[1], "%.4g"%d["value"], "cast %.3f"%d["cast_ms_per_step"], {k: round(v,3) for k,v in c.items() if k in ("nodes","leaves","instances","tlas_nodes")})
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
