import sys, numpy as np
sys.path.insert(0,'.')
from paper_1907_01995_b200 import elastic_net as en
from paper_1907_01995_b200.problems import Mode
from oracle import rac_oracle as ro
rng = np.random.default_rng(17)
for (m, n, s, mode, alpha) in [(33, 70, 9, "rac", 1.0), (400, 600, 37, "rac", 0.5),
                               (100, 513, 64, "rp", 0.2), (5, 7, 2, "rac", 1.0),
                               (70, 20, 20, "rp", 0.0), (300, 1000, 256, "rac", 0.8)]:
    X = rng.standard_normal((m, n)); y = rng.standard_normal(m)
    kw = dict(lam=0.05, alpha=alpha, gamma=0.7, block_size=s, iters=12, seed=3)
    r = ro.en_fit(X, y, mode=mode, **kw)
    g = en.fit(X, y, en.ElasticNetSpec(mode=Mode(mode), **kw), gram_mode="covariance")
    print(m, n, s, mode, np.linalg.norm(g.beta - r['beta']) / max(np.linalg.norm(r['beta']),1e-300), flush=True)
