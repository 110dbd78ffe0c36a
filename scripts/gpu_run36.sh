set -x
python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t36_pytest.log 2>&1; echo "pytest rc=$?"
RAC_EN_CS=4 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t36_pytest_cs4.log 2>&1; echo "pytest4 rc=$?"
RAC_EN_CS=8 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t36_pytest_cs8.log 2>&1; echo "pytest8 rc=$?"
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t36_bench2.log 2>&1; echo "bench2 rc=$?"
