for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_qp.py -x -q -m gpu > gpurun_out/t72_$i.log 2>&1; echo "run$i rc=$?"; done
