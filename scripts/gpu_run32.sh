set -x
python -m pytest tests/test_gpu_qp.py -x -q -m gpu > gpurun_out/t32_pytest.log 2>&1; echo "pytest rc=$?"
python scripts/prof_e2e.py 2 20 > gpurun_out/t32_e2e2.log 2>&1; echo "e2e2 rc=$?"
python scripts/prof_e2e.py 3 20 > gpurun_out/t32_e2e3.log 2>&1; echo "e2e3 rc=$?"
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu > gpurun_out/t32_bench4.log 2>&1; echo "bench4 rc=$?"
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r01_plain_cfg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r01_launch_ncu.log 2>&1; echo "launch rc=$?"
python scripts/prof_en.py 2 3 > gpurun_out/r01_en2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"en_chain" -s 1 -c 1 -o gpurun_out/r01_en_chain_cfg2 python scripts/prof_en.py 2 3 > gpurun_out/r01_en2_ncu.log 2>&1; echo "en2 rc=$?"
python scripts/prof_en.py 5 2 > gpurun_out/r01_en5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gram_kernel|en_chain" -s 0 -c 2 -o gpurun_out/r01_gram_chain_cfg5 python scripts/prof_en.py 5 2 > gpurun_out/r01_en5_ncu.log 2>&1; echo "en5 rc=$?"
python scripts/prof_svm.py 2 > gpurun_out/r01_svm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"qp_chain" -s 1 -c 1 -o gpurun_out/r01_qp_chain_cfg4 python scripts/prof_svm.py 2 > gpurun_out/r01_svm_ncu.log 2>&1; echo "svm rc=$?"
