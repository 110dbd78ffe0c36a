#!/bin/bash
# Round-2 evidence: launch lists and Nsight Compute captures of the headline kernels (one GPU).
mkdir -p gpurun_out
python scripts/prof_en.py 5 2 > gpurun_out/ev_plain5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5.csv \
    python scripts/prof_en.py 5 2 > gpurun_out/ev_l5.log 2>&1; echo "launches5 rc=$?"
ncu --set full --clock-control none --import-source on \
  -k "regex:gram_i8_kernel|i8_slice_kernel|en_chain_kernel|large_update|large_pivot|large_assemble" -s 0 -c 6 \
  -o gpurun_out/r02_cfg5 -f python scripts/prof_en.py 5 1 > gpurun_out/ev_f5.log 2>&1; echo "full5 rc=$?"
python scripts/prof_en.py 3 3 > gpurun_out/ev_plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:factor_kernel|en_cla_kernel|gram_i8_kernel" \
    -s 0 -c 3 -o gpurun_out/r02_cfg3 -f python scripts/prof_en.py 3 3 > gpurun_out/ev_f3.log 2>&1; echo "full3 rc=$?"
python scripts/prof_en.py 2 3 > gpurun_out/ev_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:en_cla_kernel" -s 1 -c 1 \
    -o gpurun_out/r02_cfg2 -f python scripts/prof_en.py 2 3 > gpurun_out/ev_f2.log 2>&1; echo "full2 rc=$?"
python scripts/prof_svm.py 2 > gpurun_out/ev_plain4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:qp_chain_kernel" -s 0 -c 1 \
    -o gpurun_out/r02_cfg4 -f python scripts/prof_svm.py 2 > gpurun_out/ev_f4.log 2>&1; echo "full4 rc=$?"
python scripts/prof_svm_strips.py 1 > gpurun_out/ev_plain4s.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:strip_kernel" -s 1 -c 1 \
    -o gpurun_out/r02_cfg4_strips -f python scripts/prof_svm_strips.py 1 > gpurun_out/ev_f4s.log 2>&1; echo "full4s rc=$?"
