# Two rays per lane (k_cast2) vs one: parity subset on the RPL2 build, then c3/c4/c5 A/B.
AGR_LIB_PATH=$PWD/build/var/r2v/libagr.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do
  bash tools/runvar.sh rpl_c3_$r "--config 3 --no-table2" base r2v r2h r2v10 r2v13
done
for c in 4 5; do
  bash tools/runvar.sh rpl_c$c "--config $c --no-table2" base r2v r2h
done
