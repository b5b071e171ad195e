# host-cast chunk count A/B (e2e) + raw pinned D2H bandwidth
python tools/pcie_d2h.py
for r in 1 2; do
for v in e2e8 e2e16 e2e32; do
  AGR_LIB_PATH=$PWD/build/var/$v/libagr.so python bench.py --config 3 --no-table2 --no-cpu-baseline --steps 10 > gpurun_out/e2e_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e2e_$v.json').read().strip().splitlines()[-1]); print('$v', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
done
done
