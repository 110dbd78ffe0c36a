timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/t18_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t18_pytest.log
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu > gpurun_out/t18_bench4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/t18_bench4.log | cut -c1-1500
