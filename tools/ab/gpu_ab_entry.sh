for c in 3 4; do
  echo "== c$c"
  bash tools/runvar.sh en_c$c "--config $c --no-table2" e0 e1 e0 e1
done
AGR_LIB_PATH=$PWD/build/var/e1/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "bvh8 or wide or c3_bench or c3_full or parts or c2_full or stereo" 2>&1 | tail -2
