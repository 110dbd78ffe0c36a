"""Where does end-to-end `fit` time go?  python scripts/prof_e2e.py CONFIG [K]"""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import _device, configs, elastic_net as en
from paper_1907_01995_b200.problems import Mode

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
case = configs.GENERATORS[cfg]()
X, y = case.X, case.y
m, n = X.shape
dev = torch.device("cuda", 0)
torch.cuda.synchronize()


def tm(label, fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{label:40s} {best * 1e3:9.2f} ms")
    return out


nb = X.nbytes
tm("pageable H2D (%.0f MB)" % (nb / 1e6), lambda: torch.from_numpy(X).to(dev))
tm("pin_memory copy", lambda: torch.from_numpy(X).pin_memory())
pinned = torch.from_numpy(X).pin_memory()
tm("pinned H2D", lambda: pinned.to(dev, non_blocking=True))
tm("_device.upload", lambda: _device.upload(X, device=dev))
rng = np.random.default_rng(0)
tm("host permutation x%d" % K, lambda: [rng.permutation(n) for _ in range(K)])
sol = en.EnSolver(m, n, case.block_size, Mode.RAC, case.lam, case.alpha, case.gamma)
gm = en.choose_gram_mode(m, n, case.block_size, K)
if gm == "covariance":
    sol.set_gram_mode("covariance")
tm("set_data (%s)" % gm, lambda: sol.set_data(X, y))
Xt = torch.from_numpy(X)
tm("stream_rows copy only", lambda: _device.stream_rows(X, 32, lambda r0, rows, d: None, device=dev))
feeder = _device.PermutationFeeder(rng, n, dev)
perms = feeder.draw(K)
tm("run K sweeps (device)", lambda: sol.run(perms, None))
tm("state", lambda: sol.state())
sol.close()
tm("EnSolver create+close", lambda: en.EnSolver(m, n, case.block_size, Mode.RAC, case.lam, case.alpha, case.gamma).close())
spec = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma, block_size=case.block_size,
                         iters=K, seed=0, tol=None)
tm("fit K sweeps (e2e)", lambda: en.fit(X, y, spec))
if case.tol is not None:
    spec2 = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma, block_size=case.block_size,
                              iters=case.iters, seed=0, tol=case.tol)
    r = tm("fit to tol (e2e)", lambda: en.fit(X, y, spec2), reps=1)
    print("sweeps", r.iterations)
