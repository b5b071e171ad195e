bash tools/profile_round.sh r02s 3 > gpurun_out/r02s_profile.log 2>&1
ls -la gpurun_out | grep r02s
