set -x
python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/n1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/n1_launches.csv python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/n1_ncu.log 2>&1
echo "rc=$?"
