set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t62_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --no-cpu > gpurun_out/t62_bench_default.log 2>&1; echo "bench rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t62_smoke.log 2>&1; echo "smoke rc=$?"
