#!/bin/bash
# Full measurement pass on the GPU box: tools/gpu_round.sh TAG
# GPU tests + smoke, every config's bench line (the default c3 line carries
# the Table-II sweep), c5 with a refit per step, the oracle arm, and the ncu
# launch lists + `--set full` captures of every config's cast.
tag=${1:-rXX}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputests.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench_c3.json 2> gpurun_out/${tag}_bench_c3.err
for c in 4 5 6; do
  timeout 600 python bench.py --config $c --no-table2 > gpurun_out/${tag}_bench_c$c.json 2> gpurun_out/${tag}_bench_c$c.err
done
timeout 600 python bench.py --config 5 --tlas-step refit --no-table2 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench_c5_refit.json 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>&1
bash tools/profile_round.sh $tag 3 4 5 6 > gpurun_out/${tag}_profile.log 2>&1
tail -2 gpurun_out/${tag}_gputests.txt
# gpurun copies back at most 64 MiB of gpurun_out/: summarise the captures on
# the box and keep only the c3 capture (plus its SASS-by-line page).
PROFILES_OUT=gpurun_out/prof_${tag} python tools/ncu_extract.py $tag > gpurun_out/${tag}_extract.txt 2>&1
cuobjdump -xelf all paper_2503_01471_b200/lib/libagr.so > /dev/null 2>&1; rm -rf /tmp/cubins; mkdir -p /tmp/cubins; mv *.cubin /tmp/cubins/ 2>/dev/null
cub=$(ls /tmp/cubins/*cast* 2>/dev/null | head -1)
[ -n "$cub" ] && python tools/sass_lines.py gpurun_out/${tag}_cast_c3.ncu-rep $cub k_cast 60 > gpurun_out/${tag}_c3_sass_lines.txt 2>&1
mkdir -p /tmp/reps; for c in 4 5 6; do mv gpurun_out/${tag}_cast_c$c.ncu-rep /tmp/reps/ 2>/dev/null; done
du -sh gpurun_out
