"""cProfile of one end-to-end fit (host arrays in, host arrays out).  python scripts/prof_fit.py CONFIG K"""
import cProfile
import pstats
import sys
import time
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import configs, elastic_net as en

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
case = configs.GENERATORS[cfg]()
spec = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma, block_size=case.block_size,
                         iters=K, seed=0, tol=None)
for _ in range(2):
    en.fit(case.X, case.y, spec)
torch.cuda.synchronize()
t0 = time.perf_counter()
en.fit(case.X, case.y, spec)
print("fit wall ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile()
pr.enable()
en.fit(case.X, case.y, spec)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
