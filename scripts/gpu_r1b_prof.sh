# Round-1 (second session) evidence: tests, bench lines of every config, launch list of
# the default bench, full captures of the lookahead chain and the factor kernel.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p2_pytest.log 2>&1; echo "pytest rc=$?"
for c in 2 1 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/p2_bench$c.log 2>&1; echo "bench$c rc=$?"
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/p2_plain_cfg2.log 2>&1 && \
RAC_PROFILE_NONCOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r01b_launches_cfg2.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/p2_launch_ncu.log 2>&1; echo "launch rc=$?"
timeout 300 python scripts/prof_en.py 2 6 > gpurun_out/p2_en2_plain.log 2>&1 && \
RAC_PROFILE_NONCOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"en_cla|factor_kernel|gram_kernel" -s 0 -c 4 -o gpurun_out/r01b_cla_factor_cfg2 -f python scripts/prof_en.py 2 6 > gpurun_out/p2_en2_ncu.log 2>&1; echo "en2 rc=$?"
