set -x
python scripts/prof_en.py 2 3 > gpurun_out/n2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sweep_inverse|gram_kernel" -s 2 -c 2 -o gpurun_out/n2_prof python scripts/prof_en.py 2 3 > gpurun_out/n2_ncu.log 2>&1
echo "rc=$?"
