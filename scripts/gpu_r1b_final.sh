# Round-1 (second session) evidence for the current state.
timeout 900 python -m pytest tests -m gpu -x -q --timeout 180 --timeout-method thread > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
for c in 2 1 3 4 5; do timeout 900 python bench.py --config $c > gpurun_out/f_bench$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/f_plain.log 2>&1 && \
RAC_PROFILE_NONCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r01c_launches_cfg2.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/f_launch_ncu.log 2>&1; echo "launch rc=$?"
timeout 300 python scripts/prof_en.py 2 7 covariance > gpurun_out/f_en2_plain.log 2>&1 && \
RAC_PROFILE_NONCOOP=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"en_cla|factor_kernel|cla_tiles|gram_kernel|gram_reduce" -s 0 -c 6 -o gpurun_out/r01c_cfg2 -f python scripts/prof_en.py 2 7 covariance > gpurun_out/f_en2_ncu.log 2>&1; echo "en2 rc=$?"
