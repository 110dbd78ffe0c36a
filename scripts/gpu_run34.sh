set -x
python -m pytest tests/test_gpu_en.py -x -q -m gpu > gpurun_out/t34_pytest.log 2>&1; echo "pytest rc=$?"
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t34_bench2.log 2>&1; echo "bench2 rc=$?"
RAC_EN_PIPE=0 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t34_bench2_nopipe.log 2>&1; echo "bench2np rc=$?"
python bench.py --config 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/t34_bench1.log 2>&1; echo "bench1 rc=$?"
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/t34_bench3.log 2>&1; echo "bench3 rc=$?"
python bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/t34_bench5.log 2>&1; echo "bench5 rc=$?"
RAC_EN_VARIANT=0 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/t34_bench2_stream.log 2>&1; echo "bench2s rc=$?"
