#!/bin/bash
# Round-2 (last session) evidence: bench line of the final state, launch list, and Nsight Compute
# captures of the two chain kernels (one GPU; numbers printed under ncu are never bench values).
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r02d_bench.log 2>&1; echo "bench rc=$?"
python scripts/prof_en.py 5 2 > gpurun_out/evd_plain5.log 2>&1 && \
  RAC_PROFILE_NONCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_launches_cfg5.csv \
    python scripts/prof_en.py 5 2 > gpurun_out/evd_l5.log 2>&1; echo "launches5 rc=$?"
RAC_PROFILE_NONCOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:en_chain_kernel" -s 0 -c 1 \
  -o gpurun_out/r02d_chain5 -f python scripts/prof_en.py 5 1 > gpurun_out/evd_c5.log 2>&1; echo "chain5 rc=$?"
python scripts/prof_svm.py 2 1.0 > gpurun_out/evd_plain4.log 2>&1 && \
  RAC_PROFILE_NONCOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:qp_chain_kernel" -s 0 -c 1 \
    -o gpurun_out/r02d_chain4 -f python scripts/prof_svm.py 2 1.0 > gpurun_out/evd_c4.log 2>&1; echo "chain4 rc=$?"
