set -x
timeout 300 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu > gpurun_out/t50_bench4.log 2>&1; echo "bench4 rc=$?"
timeout 300 python scripts/prof_svm.py 10 1.0 --trace > gpurun_out/t50_svm_trace.log 2>&1; echo "trace rc=$?"
timeout 300 python scripts/prof_svm.py 60 1.0 --trace > gpurun_out/t50_svm_trace60.log 2>&1; echo "trace rc=$?"
