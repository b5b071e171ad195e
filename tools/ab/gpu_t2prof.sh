timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/t2p_launches.csv python bench.py --table2 --t2-res 8x8 --t2-envs 2048 --t2-steps 3 --warmup 3 > gpurun_out/t2p.json 2>&1
python - <<'PY'
import csv,io,collections
lines=[l for l in open('gpurun_out/t2p_launches.csv') if l.startswith('"')]
agg=collections.defaultdict(list)
for r in csv.DictReader(io.StringIO("".join(lines))):
    agg[(r["Kernel Name"].split("(")[0][-40:], r["Metric Name"])].append(float(r["Metric Value"].replace(",","")))
for k,v in sorted(agg.items()):
    print(k, len(v), "median %.4g"%sorted(v)[len(v)//2])
PY
