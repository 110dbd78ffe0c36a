timeout 300 python -m pytest tests/test_gpu_en.py -x -q > gpurun_out/cla5_pytest.log 2>&1; echo "pytest rc=$?"
timeout 200 python bench.py --no-cpu > gpurun_out/cla5_bench.log 2>&1; echo "bench rc=$?"
timeout 200 python bench.py --no-cpu --config 1 > gpurun_out/cla5_bench1.log 2>&1; echo "bench1 rc=$?"
