"""Where do small fits spend their time right after the config-5 bench legs (host profile)."""
import cProfile
import pstats
import sys
import time

sys.argv = ["bench.py"]
sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1907_01995_b200 import configs, elastic_net as en  # noqa: E402


class A:
    steps, warmup, gram, no_cpu = 20, 5, "auto", True


peaks = bench.measured_peaks()
i8 = {"peak": 3300.0, "source": "x"}
torch.cuda.set_device(0)
c5 = configs.config5()
r5 = bench.measure_en(5, c5, A(), 1, 0, 0, peaks, 35.0, i8, False)
print("c5", r5["value"], flush=True)
del c5
torch.cuda.empty_cache()
c1 = configs.config1()
spec = en.ElasticNetSpec(lam=c1.lam, alpha=c1.alpha, gamma=c1.gamma, block_size=c1.block_size, iters=20, seed=0)
pr = cProfile.Profile()
pr.enable()
ts = []
for _ in range(6):
    t0 = time.perf_counter()
    en.fit(c1.X, c1.y, spec)
    ts.append(round(1e3 * (time.perf_counter() - t0), 2))
pr.disable()
print("c1 fits", ts, flush=True)
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
