timeout 400 python -m pytest tests/test_gpu_en.py tests/test_gpu_qp.py -x -q --timeout 120 --timeout-method thread > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?"
for c in 3 2; do timeout 300 python bench.py --no-cpu --config $c > gpurun_out/g_bench$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 300 python scripts/prof_en.py 2 7 covariance > gpurun_out/g_en2_plain.log 2>&1 && \
RAC_PROFILE_NONCOOP=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"en_cla|factor_kernel|cla_tiles|gram_kernel|gram_reduce" -s 0 -c 5 -o gpurun_out/r01c_cfg2 -f python scripts/prof_en.py 2 7 covariance > gpurun_out/g_en2_ncu.log 2>&1; echo "en2 rc=$?"
