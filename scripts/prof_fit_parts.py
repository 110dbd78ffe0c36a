"""Breakdown of one config-2 fit() through the public API (host arrays)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import _device, configs, elastic_net as en
from paper_1907_01995_b200.problems import Mode

case = configs.GENERATORS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]()
X, y = case.X, case.y
m, n = X.shape
K = 20
spec = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma, block_size=case.block_size, iters=K, seed=0)
en.fit(X, y, spec)
torch.cuda.synchronize()
for rep in range(3):
    t = [time.perf_counter()]
    sol = en.EnSolver(m, n, case.block_size, Mode.RAC, case.lam, case.alpha, case.gamma); torch.cuda.synchronize(); t.append(time.perf_counter())
    (sol.set_gram_mode("covariance") if en.choose_gram_mode(m, n, case.block_size, K) == "covariance" else None); torch.cuda.synchronize(); t.append(time.perf_counter())
    sol.set_data(X, y); torch.cuda.synchronize(); t.append(time.perf_counter())
    feeder = _device.PermutationFeeder(np.random.default_rng(0), n, sol.dev)
    perms = feeder.draw(16); p2 = feeder.draw(4); torch.cuda.synchronize(); t.append(time.perf_counter())
    sol.run(perms, None); sol.run(p2, None); torch.cuda.synchronize(); t.append(time.perf_counter())
    it = sol.progress(); b, z, xi = sol.state(); hp, hd = sol.history(K)
    out = (b.cpu().numpy(), z.cpu().numpy(), xi.cpu().numpy(), hp.cpu().numpy(), hd.cpu().numpy()); t.append(time.perf_counter())
    sol.close(); torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("create %.3f  gram_mode %.3f  set_data %.3f  perms %.3f  run %.3f  results %.3f  close %.3f  total %.3f ms" % (*d, d.sum()))
t0 = time.perf_counter(); en.fit(X, y, spec); torch.cuda.synchronize(); print("fit %.3f ms" % ((time.perf_counter() - t0) * 1e3))
