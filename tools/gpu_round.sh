timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02k_gputests.txt 2>&1
timeout 600 python bench.py --table2 > gpurun_out/r02k_table2.json 2> gpurun_out/r02k_table2.err
bash tools/profile_round.sh r02k 3 4 5 6 > gpurun_out/r02k_profile.log 2>&1
tail -3 gpurun_out/r02k_gputests.txt
