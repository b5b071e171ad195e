# compute-sanitizer over tools/sanitize_run.py: tools/gpu_sanitize.sh [TAG]
CS=/usr/local/cuda/bin/compute-sanitizer
out=gpurun_out/${1:-sanitize}.txt
for t in memcheck initcheck racecheck synccheck; do
  echo "== $t" >> $out
  timeout 1200 $CS --tool $t --kernel-name kns=agr --print-limit 20 python tools/sanitize_run.py >> $out 2>&1
  echo "exit $?" >> $out
done
grep -E '^==|ERROR SUMMARY|exit|done' $out
