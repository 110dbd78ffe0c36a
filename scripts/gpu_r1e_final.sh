timeout 900 python -m pytest tests -m gpu -x -q --timeout 180 --timeout-method thread > gpurun_out/f3_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?"
for c in 2 1 3 4 5; do timeout 900 python bench.py --config $c > gpurun_out/f3_bench$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f3_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/f3_plain.log 2>&1 && \
RAC_PROFILE_NONCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r01e_launches_cfg2.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/f3_launch_ncu.log 2>&1; echo "launch rc=$?"
