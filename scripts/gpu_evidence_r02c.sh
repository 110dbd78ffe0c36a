#!/bin/bash
# Round-2 (final state) evidence: launch list and Nsight Compute captures of the headline kernels (one GPU).
mkdir -p gpurun_out
python scripts/prof_en.py 5 2 > gpurun_out/evc_plain5.log 2>&1 && \
  RAC_PROFILE_NONCOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches_cfg5.csv \
    python scripts/prof_en.py 5 2 > gpurun_out/evc_l5.log 2>&1; echo "launches5 rc=$?"
ncu --set full --clock-control none --import-source on \
  -k "regex:gram_i8_kernel|i8_slice_kernel|en_chain_kernel|large_update|large_cw|large_pivot|large_assemble" -s 0 -c 7 \
  -o gpurun_out/r02c_cfg5 -f python scripts/prof_en.py 5 1 > gpurun_out/evc_f5.log 2>&1; echo "full5 rc=$?"
python scripts/prof_en.py 3 3 > gpurun_out/evc_plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:factor_kernel|en_cla_kernel|gram_i8_kernel" \
    -s 0 -c 3 -o gpurun_out/r02c_cfg3 -f python scripts/prof_en.py 3 3 > gpurun_out/evc_f3.log 2>&1; echo "full3 rc=$?"
