timeout 300 python scripts/prof_svm.py 60 1.0 --trace > gpurun_out/t69_svm_trace60.log 2>&1; echo "trace rc=$?"
python scripts/prof_svm.py 3 > gpurun_out/t69_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/t69_svm_launches.csv python scripts/prof_svm.py 3 > gpurun_out/t69_ncu.log 2>&1; echo "ncu rc=$?"
