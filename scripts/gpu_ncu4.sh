python scripts/prof_svm.py 2 > gpurun_out/n4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"qp_chain" -s 1 -c 1 -o gpurun_out/n4_prof python scripts/prof_svm.py 2 > gpurun_out/n4_ncu.log 2>&1
echo "rc=$?"
