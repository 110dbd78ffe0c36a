timeout 400 python -m pytest tests/test_gpu_en.py -x -q --timeout 120 --timeout-method thread > gpurun_out/t1_pytest.log 2>&1; echo "prc=$?"
timeout 400 python bench.py --no-cpu --config 5 --steps 6 --warmup 3 > gpurun_out/t1_bench5.log 2>&1; echo "b5 rc=$?"
