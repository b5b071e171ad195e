timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_gputests.txt 2>&1; tail -3 gpurun_out/t_gputests.txt
