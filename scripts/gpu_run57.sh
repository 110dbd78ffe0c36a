set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t57_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/t57_bench_default.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/t57_bench_ref.log 2>&1; echo "ref rc=$?"
export RAC_PROFILE_NONCOOP=1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r01_launches_cfg2.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/p_launch_ncu.log 2>&1; echo "launch rc=$?"
