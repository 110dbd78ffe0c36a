set -x
timeout 600 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t75_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/t75_bench5.log 2>&1; echo "bench5 rc=$?"
