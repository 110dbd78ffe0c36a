timeout 200 python bench.py --no-cpu > gpurun_out/cla3_bench.log 2>&1; echo "bench rc=$?"
timeout 300 python -m pytest tests/test_gpu_en.py -x -q > gpurun_out/cla3_pytest.log 2>&1; echo "pytest rc=$?"
