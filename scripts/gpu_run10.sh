timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/t10_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t10_pytest.log
for c in 2 1 3; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/t10_bench$c.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/t10_bench$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['stage_ms_per_sweep'], d['chain_trace'], d.get('time_to_tol'))"
done
