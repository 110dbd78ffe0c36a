"""Breakdown of one config-4 svm.train() through the public API (host arrays)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import _device, configs, svm, engine
from paper_1907_01995_b200.problems import Mode, SolverConfig
import math
case = configs.config4()
X, y = case.X, case.labels
N, d = X.shape
cfg = SolverConfig(mode=Mode.RAC, block_size=case.block_size, beta_penalty=case.beta, max_iters=20,
                   tol_primal=1e-6, tol_dual=1e-6, seed=0, fixed_iterations=True)
svm.train(X, y, case.C, svm.KernelSpec("linear"), cfg)
torch.cuda.synchronize()
dev = torch.device("cuda")
for rep in range(3):
    t = [time.perf_counter()]
    Q = svm.build_q(X, y, svm.KernelSpec("linear"), dev); torch.cuda.synchronize(); t.append(time.perf_counter())
    solver = engine.QpSolver(N, 1, case.block_size, Mode.RAC, case.beta, svm.RIDGE_REL); torch.cuda.synchronize(); t.append(time.perf_counter())
    solver.set_problem(np.full(N, -1.0), np.zeros(N), np.full(N, case.C), A=y.reshape(1, N), b=np.zeros(1), borrowed_h=Q)
    solver.set_divergence_bar(math.inf); torch.cuda.synchronize(); t.append(time.perf_counter())
    fd = _device.PermutationFeeder(np.random.default_rng(0), N, dev)
    tt = [time.perf_counter()]
    p16 = fd.draw(16); torch.cuda.synchronize(); tt.append(time.perf_counter())
    solver.run(p16, 16, 1e-6, 1e-6, True); torch.cuda.synchronize(); tt.append(time.perf_counter())
    p4 = fd.draw(4); solver.run(p4, 4, 1e-6, 1e-6, True); torch.cuda.synchronize(); tt.append(time.perf_counter())
    it, st, _ = solver.progress(); t.append(time.perf_counter())
    print("   draw16 %.1f run16 %.1f draw4+run4 %.1f ms" % tuple(np.diff(tt) * 1e3))
    x, yv, _ = solver.state(); hp, _, hd = (h.cpu().numpy() for h in solver.history(it)); z = x.cpu().numpy(); t.append(time.perf_counter())
    solver.close(); torch.cuda.synchronize(); t.append(time.perf_counter())
    b = svm._bias_from_q(Q, z, y, case.C); t.append(time.perf_counter())
    sup = z > svm.SUPPORT_THRESHOLD; m = X[sup].copy(); t.append(time.perf_counter())
    del Q; torch.cuda.synchronize(); t.append(time.perf_counter())
    dd = np.diff(t) * 1e3
    print("build_q %.1f create %.1f set_problem %.1f drive %.1f state %.1f close %.1f bias %.1f support %.1f free %.1f total %.1f ms" % (*dd, dd.sum()))
t0 = time.perf_counter(); svm.train(X, y, case.C, svm.KernelSpec("linear"), cfg); torch.cuda.synchronize(); print("train %.1f ms" % ((time.perf_counter() - t0) * 1e3))
