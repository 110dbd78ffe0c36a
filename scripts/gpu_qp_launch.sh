timeout 300 python scripts/prof_svm.py 4 1.0 > gpurun_out/j_plain.log 2>&1 && \
RAC_PROFILE_NONCOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/j_launches_cfg4.csv python scripts/prof_svm.py 4 1.0 > gpurun_out/j_ncu.log 2>&1; echo "rc=$?"
