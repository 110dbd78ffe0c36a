for t in h_only diverge; do timeout 120 python scripts/repro_hqp.py $t 2>&1 | tail -1; done
for t in h_only diverge; do RAC_QP_RESIDENT=0 timeout 120 python scripts/repro_hqp.py $t 2>&1 | tail -1; done
