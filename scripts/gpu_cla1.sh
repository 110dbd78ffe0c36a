timeout 240 python -m pytest tests/test_gpu_en.py -x -q -k "covariance or config1 or config2" > gpurun_out/cla1_pytest.log 2>&1; echo "pytest rc=$?"
timeout 200 python bench.py --no-cpu > gpurun_out/cla1_bench.log 2>&1; echo "bench rc=$?"
