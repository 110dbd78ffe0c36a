set -x
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t40_bench2.log 2>&1; echo "bench2 rc=$?"
RAC_EN_CS=8 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t40_bench2_cs8.log 2>&1; echo "bench2 rc=$?"
