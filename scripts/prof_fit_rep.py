"""Repeated fit() of one config through the public API (host arrays): wall time per call."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import configs, elastic_net as en

case = configs.GENERATORS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]()
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
spec = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma, block_size=case.block_size, iters=K, seed=0)
en.fit(case.X, case.y, spec)
torch.cuda.synchronize()
ts = []
for rep in range(6):
    t0 = time.perf_counter(); en.fit(case.X, case.y, spec); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
print("fit ms:", " ".join(f"{t:.1f}" for t in ts), " min %.1f" % min(ts))
