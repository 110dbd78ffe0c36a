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
    P = 148
    buf = (np.ctypeslib.ctypes.c_int64 * (22 * p + 2 * p * P))()
    sol.lib.rac_qp_trace(sol.h, buf, 22 * p + 2 * p * P)
    allv = np.array(buf[:], dtype=np.float64)
    tv = allv[:10 * p].reshape(p, 10) / 1e3
    dbg = allv[10 * p:14 * p].reshape(p, 4)
    arr = allv[14 * p:14 * p + 2 * p * P].reshape(p, P, 2) / 1e3
    stt = allv[14 * p + 2 * p * P:].reshape(p, 8)
    a2 = arr[:, :, 0] - arr[:, 0:1, 0]      # arrival at barrier 2 relative to CTA 0
    a1 = arr[1:, :, 1] - arr[1:, 0:1, 1]    # arrival at barrier 1 (next block) relative to CTA 0
    print("barrier2 arrival minus CTA0 (us): CTA1 %.2f  others mean %.2f max %.2f" % (
        a2[:, 1].mean(), a2[:, 2:].mean(), a2[:, 2:].max(axis=1).mean()))
    print("barrier1 arrival minus CTA0 (us): CTA1 %.2f  others mean %.2f max %.2f" % (
        a1[:, 1].mean(), a1[:, 2:].mean(), a1[:, 2:].max(axis=1).mean()))
    print("box: solves/block %.2f passes/block %.2f us in solves/block %.2f us box total/block %.2f" % (
        dbg[:, 0].mean(), dbg[:, 1].mean(), dbg[:, 2].mean() / 1e3, dbg[:, 3].mean() / 1e3))
    order = [0, 1, 2, 3, 4, 5, 6, 8, 9, 7]
    seg = np.diff(tv[:, order], axis=1)
    names = ["gather", "wait_ML", "x0", "box", "commit+prefetch", "barrier2", "hbx", "strip", "rowphase_A"]
    print("block loop us: %.1f (first S start -> last G end), per block %.2f" % (
        tv[-1, 7] - tv[0, 0], (tv[-1, 7] - tv[0, 0]) / p))
    print("per block us:", {k: round(float(v), 2) for k, v in zip(names, seg.mean(axis=0))},
          "barrier1 %.2f" % float(np.mean(tv[1:, 0] - tv[:-1, 7])))
    ns = np.maximum(stt[:, 0] * 0 + dbg[:, 0], 1)
    print("reduced solves: mean nb %.1f  mean nf %.1f  direct fraction %.2f  factor us/solve %.2f  tri-solve us/solve %.2f" % (
        stt[:, 0].sum() / max(dbg[:, 0].sum(), 1), stt[:, 1].sum() / max(dbg[:, 0].sum(), 1),
        stt[:, 2].sum() / max(dbg[:, 0].sum(), 1), stt[:, 3].sum() / 1e3 / max(dbg[:, 0].sum(), 1),
        stt[:, 4].sum() / 1e3 / max(dbg[:, 0].sum(), 1)))
