import sys, numpy as np
sys.path.insert(0,'.')
from paper_1907_01995_b200 import elastic_net as en
from paper_1907_01995_b200.problems import Mode
from oracle import rac_oracle as ro
which = sys.argv[1]
rng = np.random.default_rng(17)
cases = [(33, 70, 9, "rac", 1.0), (400, 600, 37, "rac", 0.5), (100, 513, 64, "rp", 0.2), (5, 7, 2, "rac", 1.0),
         (70, 20, 20, "rp", 0.0)]
for i, (m, n, s, mode, alpha) in enumerate(cases):
    X = rng.standard_normal((m, n)); y = rng.standard_normal(m)
    if str(i) not in which: continue
    kw = dict(lam=0.05, alpha=alpha, gamma=0.7, block_size=s, iters=12, seed=3)
    caps = {}
    r = ro.en_fit(X, y, mode=mode, **kw, on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, b.copy()))
    got = {}
    g = en.fit(X, y, en.ElasticNetSpec(mode=Mode(mode), **kw), gram_mode="covariance",
               sweep_hook=lambda k, b, z, xi: got.__setitem__(k, b))
    errs = [float(np.linalg.norm(got[k] - caps[k]) / max(np.linalg.norm(caps[k]), 1e-300)) for k in sorted(caps)]
    print(which, m, n, s, mode, ["%.1e" % e for e in errs], flush=True)
