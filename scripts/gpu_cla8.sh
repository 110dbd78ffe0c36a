timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 --timeout-method thread > gpurun_out/cla8_pytest.log 2>&1; echo "pytest rc=$?"
for c in 2 1 3; do timeout 300 python bench.py --no-cpu --config $c > gpurun_out/cla8_bench$c.log 2>&1; echo "bench$c rc=$?"; done
