timeout 600 python bench.py --no-cpu > gpurun_out/t76_bench2.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --config 3 --no-cpu > gpurun_out/t76_bench3.log 2>&1; echo "bench rc=$?"
