import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import configs, svm
from paper_1907_01995_b200.problems import Mode, SolverConfig
case = configs.config4()
X, y = case.X, case.labels
cfg = SolverConfig(mode=Mode.RAC, block_size=case.block_size, beta_penalty=case.beta, max_iters=20,
                   tol_primal=1e-6, tol_dual=1e-6, seed=0, fixed_iterations=True)
for rep in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    svm.train(X, y, case.C, svm.KernelSpec("linear"), cfg)
    torch.cuda.synchronize(); print("train %d: %.1f ms  torch reserved %.2f GB" % (rep, (time.perf_counter() - t0) * 1e3, torch.cuda.memory_reserved()/1e9))
