"""Host-side profile of repeated small fits (config 1): wall time per fit and the top functions."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch
from paper_1907_01995_b200 import configs, elastic_net as en

c = configs.config1()
spec = en.ElasticNetSpec(lam=c.lam, alpha=c.alpha, gamma=c.gamma, block_size=c.block_size, iters=20, seed=0)
for _ in range(3):
    en.fit(c.X, c.y, spec)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    en.fit(c.X, c.y, spec)
    ts.append(time.perf_counter() - t0)
print("fit ms:", [round(1e3 * t, 2) for t in ts])
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    en.fit(c.X, c.y, spec)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
