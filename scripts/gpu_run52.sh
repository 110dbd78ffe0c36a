set -x
timeout 300 python scripts/prof_svm.py 60 1.0 --trace > gpurun_out/t52_svm_trace60.log 2>&1; echo "trace rc=$?"
timeout 600 python -m pytest tests/test_gpu_qp.py -x -q -m gpu > gpurun_out/t52_pytest.log 2>&1; echo "pytest rc=$?"
