for c in 3 4 5; do
  echo "== c$c"
  bash tools/runvar.sh fm_c$c "--config $c --no-table2" f0 f1
done
AGR_LIB_PATH=$PWD/build/var/f1/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "bvh8 or wide or c3_bench or c2_full or axis_aligned or scaled or c4_full or c5_sampled or sensor_on" 2>&1 | tail -3
