#!/usr/bin/env python
"""Per-launch times (us) of the last bench step in an ncu launch list:
  tools/launch_breakdown.py gpurun_out/X_launches_c6.csv [first-kernel-of-step]"""
import csv
import io
import sys

path = sys.argv[1]
first = sys.argv[2] if len(sys.argv) > 2 else "k_seg_of"
lines = [l for l in open(path) if l.startswith('"')]
rows = [(r["Kernel Name"].split("(")[0].replace("agr::<unnamed>::", ""), float(r["Metric Value"].replace(",", "")))
        for r in csv.DictReader(io.StringIO("".join(lines))) if r["Metric Name"] == "gpu__time_duration.sum"]
idx = [i for i, (k, _) in enumerate(rows) if k == first]
last = rows[idx[-1]:] if idx else rows
tot = 0.0
for k, t in last:
    print("%-44s %9.1f us" % (k[:44], t / 1000))
    tot += t
print("total %.3f ms" % (tot / 1e6))
