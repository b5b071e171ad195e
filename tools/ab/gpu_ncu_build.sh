# ncu --set full of the c6 BLAS build kernels (creation-time batch = the per-step batch)
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
   -k "regex:k_fit|k_reach4|k_write4$|k_pack_tris|k_karras|k_tri_prep|k_rs_scatter" -c 7 -f -o gpurun_out/c6b_build \
   python bench.py --config 6 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2 > gpurun_out/c6b_ncu.log 2>&1
tail -3 gpurun_out/c6b_ncu.log
