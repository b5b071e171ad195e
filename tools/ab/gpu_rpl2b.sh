bash tools/runvar.sh rplb_c3 "--config 3 --no-table2" base r2v r2h
bash tools/runvar.sh rplb_c4 "--config 4 --no-table2" base r2v
bash tools/ab/gpu_rpl2_prof.sh
