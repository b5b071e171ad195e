#!/bin/bash
# usage: tools/profile_round.sh TAG [configs...]   (run on the GPU box via gpurun)
# 1) launch list of one bench step (gpu__time_duration per launch, cold and
#    serialised: shares only), 2) one `ncu --set full` capture of k_cast per
#    config.  Outputs under gpurun_out/; tools/ncu_extract.py summarises them.
tag=$1; shift
cfgs=${@:-3 4 5 6}
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-counters --no-table2"
for c in $cfgs; do
  timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_launches_c$c.csv $B --config $c > /dev/null 2>&1
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_cast \
      --launch-skip 3 --launch-count 1 -f -o gpurun_out/${tag}_cast_c$c \
      $B --config $c > gpurun_out/${tag}_ncu_c$c.log 2>&1
done
ls -la gpurun_out/ | grep $tag
