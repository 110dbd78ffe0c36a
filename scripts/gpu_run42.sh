set -x
python -m pytest tests -x -q -m gpu > gpurun_out/t42_pytest.log 2>&1; echo "pytest rc=$?"
for c in 1 2 3 5; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/t42_bench$c.log 2>&1; echo "bench$c rc=$?"; done
python bench.py --config 4 --steps 20 --warmup 5 --no-cpu > gpurun_out/t42_bench4.log 2>&1; echo "bench4 rc=$?"
