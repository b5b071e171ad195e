AGR_LIB_PATH=$PWD/build/var/pf/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "c6 or lane or update or wide_tile" 2>&1 | tail -2
for r in 1 2; do for v in pf0 pf; do bash tools/runab.sh l2pf_${v}_$r $v "--config 6 --no-table2"; done; done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 --config 6"
AGR_LIB_PATH=$PWD/build/var/pf/libagr.so timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:k_cast \
   --launch-skip 3 --launch-count 1 -f -o gpurun_out/l2pf_c6 $B > gpurun_out/l2pf_ncu.log 2>&1
tail -1 gpurun_out/l2pf_ncu.log
