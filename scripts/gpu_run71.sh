timeout 300 python -m pytest tests/test_gpu_qp.py -x -q -m gpu -k "solve_matches_reference" > gpurun_out/t71_a.log 2>&1; echo "a rc=$?"
RAC_QP_PF=0 timeout 300 python -m pytest tests/test_gpu_qp.py -x -q -m gpu -k "solve_matches_reference" > gpurun_out/t71_b.log 2>&1; echo "b rc=$?"
python - > gpurun_out/t71_c.log 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np
g=np.load('tests/golden/qp_small.npz')
print([k for k in g.keys() if k.startswith('box_rac')][:20])
for k in g.keys():
    if k.startswith('box_rac') and g[k].ndim<=2: print(k, g[k].shape)
PY
