set -x
timeout 300 python scripts/prof_svm.py 60 1.0 --trace > gpurun_out/t63_svm_trace60.log 2>&1; echo "trace rc=$?"
