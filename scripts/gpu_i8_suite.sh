#!/bin/bash
# full GPU suite + benches of the configs the covariance Gram touches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/i8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i8_pytest.log
for c in 2 3 1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/i8_bench$c.log 2>&1
done
