#!/usr/bin/env python
"""Summarise ncu captures (run here, after gpurun brought them back):
  tools/ncu_extract.py TAG [configs...]
reads gpurun_out/TAG_cast_cN.ncu-rep (`--set full`) and
gpurun_out/TAG_launches_cN.csv (per-launch gpu__time_duration), writes
profiles/TAG_cast_cN_ncu_metrics.json and profiles/TAG_launches_cN.csv (or
under $PROFILES_OUT), and
prints each kernel's share of the launch list."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
    "l1tex__t_sector_hit_rate.pct", "launch__block_size", "launch__grid_size",
    "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "sass__inst_executed_local_loads",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__warps_eligible.avg.per_cycle_active",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum",
]


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: [v, u] for h, u, v in zip(hdr, units, vals)}


def shares(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"].split("(")[0], float(r["Metric Value"].replace(",", ""))))
    tot = sum(t for _, t in rows) or 1.0
    agg = {}
    for k, t in rows:
        agg[k] = agg.get(k, 0.0) + t
    return {k: round(100 * v / tot, 2) for k, v in sorted(agg.items(), key=lambda x: -x[1])}


def main():
    tag = sys.argv[1]
    cfgs = sys.argv[2:] or ["3", "4", "5", "6"]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.environ.get("PROFILES_OUT", os.path.join(root, "profiles"))
    os.makedirs(out, exist_ok=True)
    for c in cfgs:
        rep = os.path.join(root, "gpurun_out", f"{tag}_cast_c{c}.ncu-rep")
        if os.path.exists(rep):
            m = raw(rep)
            d = {k: m[k] for k in KEYS if k in m}
            d["kernel"] = m.get("Kernel Name", ["?"])[0]
            with open(os.path.join(out, f"{tag}_cast_c{c}_ncu_metrics.json"), "w") as f:
                json.dump(d, f, indent=1)
            print(f"c{c}", {k.split("__")[-1][:40]: v[0] for k, v in d.items() if k != "kernel"})
        lc = os.path.join(root, "gpurun_out", f"{tag}_launches_c{c}.csv")
        if os.path.exists(lc):
            shutil.copy(lc, os.path.join(out, f"{tag}_launches_c{c}.csv"))
            print(f"c{c} launch shares %:", shares(lc))


if __name__ == "__main__":
    main()
