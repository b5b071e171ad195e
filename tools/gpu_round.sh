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
