set -x
for c in 1 2 3 5 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/b_cfg$c.log 2>&1; echo "cfg $c rc=$?"; tail -2 gpurun_out/b_cfg$c.log | cut -c1-3000
done
