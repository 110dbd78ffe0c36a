# Re-entry check: GPU tests, smoke, default bench.
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c1_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/c1_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/c1_bench_ref.log 2>&1; echo "ref rc=$?"
