timeout 300 python scripts/prof_en.py 5 2 blocks > gpurun_out/i_en5_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"en_chain_kernel" -s 0 -c 1 -o gpurun_out/r01d_chain1t_cfg5 -f python scripts/prof_en.py 5 2 blocks > gpurun_out/i_en5_ncu.log 2>&1; echo "en5 rc=$?"
