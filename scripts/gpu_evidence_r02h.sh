#!/bin/bash
# Round-2 final state: launch list (config 5) and Nsight Compute captures of the headline's kernels.
mkdir -p gpurun_out
python scripts/prof_en.py 5 2 > gpurun_out/evh_plain5.log 2>&1 && \
  RAC_PROFILE_NONCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches_cfg5.csv \
    python scripts/prof_en.py 5 2 > gpurun_out/evh_l5.log 2>&1; echo "launches5 rc=$?"
RAC_PROFILE_NONCOOP=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:en_chain_kernel|gram_i8_kernel|i8_slice_kernel|large_update" -s 0 -c 12 \
  -o gpurun_out/r02h_cfg5 -f python scripts/prof_en.py 5 1 > gpurun_out/evh_c5.log 2>&1; echo "full5 rc=$?"
