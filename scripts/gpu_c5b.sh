timeout 400 python bench.py --no-cpu --config 5 --steps 6 --warmup 3 > gpurun_out/c5b_bench5.log 2>&1; echo "b5 rc=$?"
