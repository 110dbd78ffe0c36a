set -x
python scripts/prof_svm.py 3 > gpurun_out/t53_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/t53_svm_launches.csv python scripts/prof_svm.py 3 > gpurun_out/t53_ncu.log 2>&1; echo "ncu rc=$?"
