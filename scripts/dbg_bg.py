import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import elastic_net as en
rng = np.random.default_rng(31)
order = sys.argv[1:]
shapes = [(400, 700, 150), (9000, 520, 130)]
data = {sh: (rng.standard_normal((sh[0], sh[1])),) for sh in shapes}
for ing in order:
    for (m, n, s) in shapes:
        X = data[(m, n, s)][0]; y = X[:, 0]
        kw = dict(lam=0.05, alpha=0.6, gamma=1.0, block_size=s, iters=6, seed=8)
        Xin = X if ing == "host" else torch.from_numpy(X).cuda()
        try:
            g = en.fit(Xin, y, en.ElasticNetSpec(**kw), gram_mode="blocks")
            print(ing, m, n, s, "ok", flush=True)
        except Exception as e:
            print(ing, m, n, s, "ERR", str(e)[:120], flush=True)
