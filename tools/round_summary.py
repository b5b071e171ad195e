#!/usr/bin/env python
"""profiles/TAG_summary.md from the TAG measurement pass (tools/gpu_round.sh TAG,
then tools/ncu_extract.py TAG): tools/round_summary.py TAG "free text"."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
note = sys.argv[2] if len(sys.argv) > 2 else ""
P = lambda f: os.path.join(ROOT, "profiles", f)


def line(f):
    return json.loads(open(P(f)).read().strip().splitlines()[-1])


rows = []
for c, f in ((3, f"{tag}_bench_c3.json"), (4, f"{tag}_bench_c4.json"), (5, f"{tag}_bench_c5.json"),
             ("5 refit", f"{tag}_bench_c5_refit.json"), (6, f"{tag}_bench_c6.json")):
    if not os.path.exists(P(f)):
        continue
    d = line(f)
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    cb = d.get("cpu_baseline") or {}
    ev = f"{e['value'] / 1e9:.2f} G" if e.get("value") else "(not run)"
    cv = f"{cb['value']:.0f}" if cb.get("value") else "(not run)"
    rows.append(f"| c{c} | {d['value'] / 1e9:.2f} G | {d['ms_per_step']:.2f} ({d['update_ms_per_step']:.3f} + "
                f"{d['cast_ms_per_step']:.2f}) | {ev} | {r.get('frac', 0):.3f} | {cv} |")
keys = [("duration (ms)", "gpu__time_duration.sum"), ("warp instructions", "smsp__inst_executed.sum"),
        ("issue slots busy %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("ALU pipe %", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        ("FMA pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("SIMD threads/instr", "smsp__thread_inst_executed_per_inst_executed.ratio"),
        ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("L2 hit %", "lts__t_sector_hit_rate.pct"), ("L1 hit %", "l1tex__t_sector_hit_rate.pct"),
        ("stall long_scoreboard", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
        ("stall wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"),
        ("stall not_selected", "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"),
        ("DRAM read", "dram__bytes_read.sum"), ("DRAM write", "dram__bytes_write.sum")]
m = {c: json.load(open(P(f"{tag}_cast_c{c}_ncu_metrics.json"))) for c in (3, 4, 5, 6)
     if os.path.exists(P(f"{tag}_cast_c{c}_ncu_metrics.json"))}
tab = ["| | " + " | ".join(f"c{c}" for c in m) + " |", "|---|" + "---|" * len(m)]
for name, k in keys:
    vals = []
    for c in m:
        v = m[c].get(k, ["-", ""])
        try:
            x = float(v[0])
            s = f"{x:.4g}"
        except ValueError:
            s = v[0]
        vals.append(s + (" " + v[1] if k.startswith("dram") else ""))
    tab.append(f"| {name} | " + " | ".join(vals) + " |")
tests = open(P(f"{tag}_gputests.txt")).read().strip().splitlines()[-1] if os.path.exists(P(f"{tag}_gputests.txt")) else "?"
txt = f"""# {tag} — measurement pass

One B200 (`tools/gpu_round.sh {tag}`): smoke (`{tag}_smoke.txt`), GPU tests
(`{tests}`), every config's bench line (`{tag}_bench_*.json`; the c3
line carries the Table-II sweep under `table2`), the oracle arm
(`{tag}_bench_reference.json`), ncu launch lists (`{tag}_launches_c*.csv`) and
`--set full` captures of every cast (`{tag}_cast_c*_ncu_metrics.json`).

| config | rays/s | ms/step (update + cast) | e2e rays/s | ALU frac | CPU oracle rays/s (16 cores) |
|---|---|---|---|---|---|
""" + "\n".join(rows) + "\n\nncu of the casts (c6: one ray per lane):\n\n" + "\n".join(tab) + "\n\n" + note + "\n"
open(P(f"{tag}_summary.md"), "w").write(txt)
print(txt)
