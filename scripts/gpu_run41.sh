set -x
python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t41_pytest.log 2>&1; echo "pytest rc=$?"
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t41_bench2.log 2>&1; echo "bench2 rc=$?"
RAC_EN_CS=2 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t41_bench2_cs2.log 2>&1; echo "bench2 rc=$?"
python bench.py --config 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/t41_bench1.log 2>&1; echo "bench1 rc=$?"
RAC_EN_CS=2 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/t41_bench1_cs2.log 2>&1; echo "bench1 rc=$?"
