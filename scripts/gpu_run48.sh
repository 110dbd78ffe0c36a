set -x
timeout 600 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t48_pytest.log 2>&1; echo "pytest rc=$?"
for c in 1 2 3; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/t48_bench$c.log 2>&1; echo "bench$c rc=$?"; done
