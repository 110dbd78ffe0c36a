set -x
timeout 900 python -m pytest tests/test_gpu_en.py -x -q -m gpu -k "not library_loaded" > gpurun_out/t2_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/t2_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/t2_bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/t2_bench.log
