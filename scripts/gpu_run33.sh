set -x
python scripts/prof_e2e.py 2 20 > gpurun_out/t33_e2e2.log 2>&1; echo "e2e2 rc=$?"
python scripts/prof_fit.py 2 20 > gpurun_out/t33_fit2.log 2>&1; echo "fit2 rc=$?"
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t33_bench2.log 2>&1; echo "bench2 rc=$?"
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/t33_bench3.log 2>&1; echo "bench3 rc=$?"
export RAC_PROFILE_NONCOOP=1
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r01_plain_cfg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r01_launch_ncu.log 2>&1; echo "launch rc=$?"
python scripts/prof_en.py 2 3 > gpurun_out/r01_en2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"en_chain" -s 1 -c 1 -o gpurun_out/r01_en_chain_cfg2 python scripts/prof_en.py 2 3 > gpurun_out/r01_en2_ncu.log 2>&1; echo "en2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"gram_kernel" -s 1 -c 1 -o gpurun_out/r01_gram_cfg2 python scripts/prof_en.py 2 3 > gpurun_out/r01_gram2_ncu.log 2>&1; echo "gram2 rc=$?"
