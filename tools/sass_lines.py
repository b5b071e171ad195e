#!/usr/bin/env python
"""Aggregate an ncu SASS source page by CUDA source line.
  tools/sass_lines.py REPORT.ncu-rep KERNEL.cubin KERNEL_SUBSTR [top]
The cubin must be the one profiled (same build, compiled with -lineinfo);
nvdisasm -g maps SASS addresses to file:line."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ia, iex, ist, ith = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Thread Instructions Executed")
prof = {}
for r in rows[1:]:
    try:
        prof[int(r[ia], 16)] = (float(r[iex] or 0), float(r[ist] or 0), float(r[ith] or 0))
    except (ValueError, IndexError):
        pass
dis = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# find the kernel's function section
cur_fn, cur_line, in_fn = None, None, False
addr_line = {}
for l in dis.splitlines():
    if l.startswith("//-----") and ".text." in l:
        in_fn = kname in l
    m2 = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m2:
        cur_line = (m2.group(1).split("/")[-1], int(m2.group(2)))
        continue
    m3 = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m3 and in_fn:
        addr_line[int(m3.group(1), 16)] = cur_line
base = min(prof) if prof else 0  # runtime addresses: the kernel starts at offset 0
prof = {a - base: v for a, v in prof.items()}
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
tot = [0.0, 0.0, 0.0]
for a, (ex, st, th) in prof.items():
    key = addr_line.get(a, ("?", 0))
    for k, v in enumerate((ex, st, th)):
        agg[key][k] += v
        tot[k] += v
print(f"mapped {sum(1 for a in prof if a in addr_line)} / {len(prof)} SASS addresses; "
      f"warp instr {tot[0]:.4g}, stall samples {tot[1]:.4g}")
src = {}
for key, (ex, st, th) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    f, ln = key
    print(f"{f}:{ln:<5} instr {100*ex/tot[0]:5.1f}%  stall {100*st/max(tot[1],1):5.1f}%  thr/instr {th/max(ex,1):5.1f}")
