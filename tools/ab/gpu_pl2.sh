timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "c6 or lane or mode or wide_tile or schedule or update or host" 2>&1 | tail -2
bash tools/runab.sh pl2_c6 pl0 "--config 6 --no-table2"
for v in pl16 pl8 pl24 pl16s4 pl16s16; do bash tools/runab.sh pl2_c6_${v} $v "--config 6 --no-table2"; done
