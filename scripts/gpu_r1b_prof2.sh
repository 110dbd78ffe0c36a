timeout 120 python scripts/cla_trace.py 2 > gpurun_out/cla_trace2.log 2>&1; echo "trace rc=$?"
timeout 300 python scripts/prof_en.py 2 6 covariance > gpurun_out/p3_en2_plain.log 2>&1 && \
RAC_PROFILE_NONCOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"en_cla|factor_kernel|cla_tiles" -s 0 -c 3 -o gpurun_out/r01b_cla_factor_cfg2 -f python scripts/prof_en.py 2 6 covariance > gpurun_out/p3_en2_ncu.log 2>&1; echo "en2 rc=$?"
