"""Small driver for ncu: RAC sweeps of BASELINE config 4 (linear SVM dual) through the native QP engine."""
import math
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import _device, configs, svm
from paper_1907_01995_b200.engine import QpSolver
from paper_1907_01995_b200.problems import Mode

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
case = configs.config4(scale=scale)
X, y = case.X, case.labels
N = X.shape[0]
dev = _device.require_cuda(0)
Q = svm.build_q(X, y, svm.KernelSpec("linear"), dev)
sol = QpSolver(N, 1, case.block_size, Mode.RAC, case.beta, svm.RIDGE_REL)
sol.set_problem(np.full(N, -1.0), np.zeros(N), np.full(N, case.C), A=y.reshape(1, N), b=np.zeros(1), borrowed_h=Q)
sol.set_divergence_bar(math.inf)
perms = _device.PermutationFeeder(np.random.default_rng(0), N, dev).draw(sweeps)
trace = "--trace" in sys.argv
if trace:
    sol.lib.rac_qp_set_trace(sol.h, 1)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
sol.run(perms, sweeps, 1e-6, 1e-6, True)
t1.record()
torch.cuda.synchronize()
print("ok", sol.progress(), "ms/sweep", t0.elapsed_time(t1) / sweeps)
if trace:
    p = sol.p
    buf = (np.ctypeslib.ctypes.c_int64 * (12 * p))()
    sol.lib.rac_qp_trace(sol.h, buf, 12 * p)
    allv = np.array(buf[:], dtype=np.float64)
    tv = allv[:8 * p].reshape(p, 8) / 1e3
    dbg = allv[8 * p:].reshape(p, 4)
    print("box: solves/block %.2f passes/block %.2f us in solves/block %.2f us box total/block %.2f" % (
        dbg[:, 0].mean(), dbg[:, 1].mean(), dbg[:, 2].mean() / 1e3, dbg[:, 3].mean() / 1e3))
    seg = np.diff(tv, axis=1)
    names = ["gather", "wait_ML", "x0", "box", "commit+prefetch", "barrier2", "G"]
    print("per block us:", {k: round(float(v), 2) for k, v in zip(names, seg.mean(axis=0))},
          "barrier1 %.2f" % float(np.mean(tv[1:, 0] - tv[:-1, 7])))
