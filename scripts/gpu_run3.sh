set -x
timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/t3_pytest.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/t3_pytest.log
