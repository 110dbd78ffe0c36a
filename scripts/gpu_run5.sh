set -x
timeout 900 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t5_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/t5_pytest.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t5_bench2.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/t5_bench2.log | cut -c1-1800
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/t5_bench1.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/t5_bench1.log | cut -c1-1800
