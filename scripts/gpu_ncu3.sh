python scripts/prof_en.py 2 3 > gpurun_out/n3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"factor_kernel" -s 1 -c 1 -o gpurun_out/n3_prof python scripts/prof_en.py 2 3 > gpurun_out/n3_ncu.log 2>&1
echo "rc=$?"
