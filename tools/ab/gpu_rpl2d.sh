bash tools/runvar.sh rpld_c3 "--config 3 --no-table2" base r2v10 r2h10
bash tools/runvar.sh rpld_c4 "--config 4 --no-table2" base r2v10 r2h10
bash tools/runvar.sh rpld_c5 "--config 5 --no-table2" base r2v10 r2h10
