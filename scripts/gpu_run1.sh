set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_en.py -x -q -m gpu -k "not library_loaded" > gpurun_out/t1_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/t1_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/t1_smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/t1_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/t1_bench.log 2>&1; echo "bench rc=$?"; tail -5 gpurun_out/t1_bench.log
