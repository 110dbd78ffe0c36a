set -x
python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t37_pytest.log 2>&1; echo "pytest rc=$?"
RAC_EN_CS=4 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t37_pytest_cs4.log 2>&1; echo "pytest4 rc=$?"
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t37_bench2.log 2>&1; echo "bench2 rc=$?"
RAC_EN_CS=4 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t37_bench2_cs4.log 2>&1; echo "bench2 rc=$?"
python bench.py --config 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/t37_bench1.log 2>&1; echo "bench1 rc=$?"
