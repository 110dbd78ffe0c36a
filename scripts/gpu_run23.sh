timeout 300 compute-sanitizer --tool memcheck python scripts/repro_hqp.py h_only > gpurun_out/memcheck.log 2>&1; echo "rc=$?"
grep -E "Invalid|at |by thread|Address|ERROR SUMMARY" gpurun_out/memcheck.log | head -30
