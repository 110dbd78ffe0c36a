set -x
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t38_bench2.log 2>&1; echo "bench2 rc=$?"
python bench.py --config 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/t38_bench1.log 2>&1; echo "bench1 rc=$?"
