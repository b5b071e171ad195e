for r in 1 2 3; do for v in pf0 pf pfn; do bash tools/runab.sh l2pf2_${v}_$r $v "--config 6 --no-table2 --no-counters"; done; done
