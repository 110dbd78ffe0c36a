"""Time the covariance Gram G = X'X/m formation (one fit's one-time cost) for a BASELINE config."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import _device, configs, elastic_net as en
from paper_1907_01995_b200.problems import Mode

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
case = configs.GENERATORS[cfg]()
m, n = case.X.shape
sol = en.EnSolver(m, n, case.block_size, Mode.RAC, case.lam, case.alpha, case.gamma)
sol.set_gram_mode("covariance")
sol.set_data(case.X, case.y)
feed = _device.PermutationFeeder(np.random.default_rng(0), n, sol.dev)
sol.run(feed.draw(2), None)
torch.cuda.synchronize()
res = []
for rep in range(5):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    p1, p2 = feed.draw(1), feed.draw(1)
    torch.cuda.synchronize()
    e[0].record()
    sol.set_gram_mode("covariance")        # G re-formed by the next run
    sol.run(p1, None)
    e[1].record()
    sol.run(p2, None)
    e[2].record()
    torch.cuda.synchronize()
    res.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
r = np.array(res)[1:]
print(f"cfg{cfg} m={m} n={n}: G + 1 sweep {r[:,0].mean():.3f} ms, 1 sweep {r[:,1].mean():.3f} ms, "
      f"G ~ {r[:,0].mean() - r[:,1].mean():.3f} ms ({m * n * (n + 1) / (r[:,0].mean() - r[:,1].mean()) / 1e9:.1f} TFLOP/s)")
