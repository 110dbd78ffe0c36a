timeout 300 python bench.py --no-cpu --config 5 --steps 6 --warmup 3 > gpurun_out/rp_bench5.log 2>&1; echo "b5 rc=$?"
timeout 300 python bench.py --no-cpu --config 4 > gpurun_out/rp_bench4.log 2>&1; echo "b4 rc=$?"
timeout 500 python -m pytest tests -m gpu -x -q --timeout 120 --timeout-method thread > gpurun_out/rp_pytest.log 2>&1; echo "prc=$?"
