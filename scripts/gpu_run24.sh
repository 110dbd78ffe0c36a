for t in box_rac h_only diverge free_cyclic; do timeout 120 python scripts/repro_hqp.py $t 2>&1 | tail -1; done
