tag=r02x
timeout 600 python bench.py --config 4 --no-table2 > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err
bash tools/profile_round.sh $tag 4 > gpurun_out/${tag}_profile4.log 2>&1
PROFILES_OUT=gpurun_out/prof_${tag} python tools/ncu_extract.py $tag 4 > gpurun_out/${tag}_extract4.txt 2>&1
rm -f gpurun_out/${tag}_cast_c4.ncu-rep
