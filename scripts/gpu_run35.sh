set -x
python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t35_pytest.log 2>&1; echo "pytest rc=$?"
for cs in 2 4 8; do RAC_EN_CS=$cs python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t35_bench2_cs$cs.log 2>&1; echo "bench2 cs=$cs rc=$?"; done
RAC_EN_CS=4 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t35_pytest_cs4.log 2>&1; echo "pytest4 rc=$?"
RAC_EN_CS=8 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t35_pytest_cs8.log 2>&1; echo "pytest8 rc=$?"
python bench.py --config 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/t35_bench1.log 2>&1; echo "bench1 rc=$?"
