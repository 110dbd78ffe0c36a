set -x
timeout 900 python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t74_pytest.log 2>&1; echo "pytest rc=$?"
for c in 2 3; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/t74_bench$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 300 python scripts/prof_e2e.py 2 20 > gpurun_out/t74_e2e2.log 2>&1
