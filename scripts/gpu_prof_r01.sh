# Round-1 profile set: launch list of the default bench + full captures of the dominant kernels.
set -x
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/p_plain_cfg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01_launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/p_launch_ncu.log 2>&1; echo "launch rc=$?"
python scripts/prof_en.py 2 3 > gpurun_out/p_en2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"en_cov|factor_kernel" -s 2 -c 2 -o gpurun_out/r01_cov_factor_cfg2 -f python scripts/prof_en.py 2 3 > gpurun_out/p_en2_ncu.log 2>&1; echo "en2 rc=$?"
python scripts/prof_en.py 3 2 > gpurun_out/p_en3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"en_cov|gram_kernel" -s 0 -c 2 -o gpurun_out/r01_gram_cov_cfg3 -f python scripts/prof_en.py 3 2 > gpurun_out/p_en3_ncu.log 2>&1; echo "en3 rc=$?"
python scripts/prof_en.py 5 2 > gpurun_out/p_en5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gram_kernel|en_chain|large_update" -s 0 -c 3 -o gpurun_out/r01_gram_chain_cfg5 -f python scripts/prof_en.py 5 2 > gpurun_out/p_en5_ncu.log 2>&1; echo "en5 rc=$?"
