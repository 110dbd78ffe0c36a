timeout 600 python scripts/prof_svm.py 3 1.0 --trace 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_qp.py -x -q -m gpu 2>&1 | tail -2
