"""Small fits (config 1) timed before and after a large fit (config 5) in the same process."""
import sys
import time

sys.path.insert(0, ".")
import torch
from paper_1907_01995_b200 import configs, elastic_net as en


def time_fits(case, iters, reps=5):
    spec = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma, block_size=case.block_size,
                             iters=iters, seed=0)
    en.fit(case.X, case.y, spec)
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        en.fit(case.X, case.y, spec)
        out.append(round(1e3 * (time.perf_counter() - t0), 2))
    return out


c1 = configs.config1()
print("config 1 fresh:", time_fits(c1, 20), flush=True)
c5 = configs.config5()
print("config 5:", time_fits(c5, 20, 2), flush=True)
print("config 1 after config 5:", time_fits(c1, 20), flush=True)
print("pool:", [(k[0][:3], k[1]) for k in en._POOL], flush=True)
en.release_pool()
print("config 1 after release_pool:", time_fits(c1, 20), flush=True)
