set -x
timeout 600 python -m pytest tests/test_gpu_qp.py -x -q -m gpu > gpurun_out/t73_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python scripts/prof_svm.py 60 1.0 --trace > gpurun_out/t73_svm_trace60.log 2>&1; echo "trace rc=$?"
timeout 300 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu > gpurun_out/t73_bench4.log 2>&1; echo "bench4 rc=$?"
