#!/usr/bin/env python
"""profiles/cast_ncu.json from one measurement pass's `ncu --set full`
captures of k_cast (profiles/TAG_cast_cN_ncu_metrics.json, written by
tools/ncu_extract.py): per config the DRAM traffic of one launch and the
counters the north star names (L2 hit rate, FP32-pipe utilisation, issue
activity).  bench.py copies the entry of its config into the JSON line
(roofline.traffic, roofline.ncu).   tools/cast_ncu_summary.py TAG"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}
out = {"source": f"ncu --set full --clock-control none -k regex:k_cast, one launch per config "
                 f"(profiles/{tag}_cast_cN_ncu_metrics.json); traffic = dram__bytes_read.sum + "
                 f"dram__bytes_write.sum (bytes)"}
for c in (3, 4, 5, 6):
    p = os.path.join(ROOT, "profiles", f"{tag}_cast_c{c}_ncu_metrics.json")
    if not os.path.exists(p):
        continue
    m = json.load(open(p))
    val = lambda k: float(m[k][0])
    b = lambda k: val(k) * UNIT[m[k][1]]
    ms = val("gpu__time_duration.sum") * (1e-3 if m["gpu__time_duration.sum"][1] == "us" else 1.0)
    traffic = b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
    out[f"c{c}"] = {
        "kernel": m.get("kernel"),
        "traffic": int(traffic),
        "kernel_ms_ncu": ms,
        "dram_gbs_ncu": traffic / (ms / 1e3) / 1e9,
        "l2_hit_pct": val("lts__t_sector_hit_rate.pct"),
        "l1_hit_pct": val("l1tex__t_sector_hit_rate.pct"),
        "fma_pipe_pct": val("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": val("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "simd_threads_per_inst": val("smsp__thread_inst_executed_per_inst_executed.ratio"),
        "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
    }
json.dump(out, open(os.path.join(ROOT, "profiles", "cast_ncu.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
