for c in 3 2 1; do timeout 300 python bench.py --no-cpu --config $c > gpurun_out/w_bench$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 400 python -m pytest tests/test_gpu_en.py -x -q --timeout 120 --timeout-method thread > gpurun_out/w_pytest.log 2>&1; echo "prc=$?"
