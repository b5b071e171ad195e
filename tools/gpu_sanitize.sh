CS=/usr/local/cuda/bin/compute-sanitizer
for t in memcheck initcheck racecheck synccheck; do
  echo "== $t" >> gpurun_out/sanitize.txt
  timeout 1200 $CS --tool $t --kernel-name kns=agr --print-limit 20 python tools/sanitize_run.py >> gpurun_out/sanitize.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize.txt
done
grep -E '^==|ERROR SUMMARY|exit|done' gpurun_out/sanitize.txt
