import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1907_01995_b200 import engine
from paper_1907_01995_b200.problems import Mode, QpProblem, SolverConfig
g = dict(np.load('tests/golden/qp_small.npz'))
tag = sys.argv[1] if len(sys.argv) > 1 else 'h_only'
bs, beta, iters, tp, td, seed, fixed = g[f"{tag}_params"]
prob = QpProblem(c=g[f"{tag}_c"], H=g.get(f"{tag}_H"), A=g.get(f"{tag}_A"), b=g.get(f"{tag}_b"),
                 lower=g[f"{tag}_lower"], upper=g[f"{tag}_upper"])
cfg = SolverConfig(mode=Mode(str(g[f"{tag}_mode"])), block_size=int(bs), beta_penalty=float(beta),
                   max_iters=int(iters), tol_primal=float(tp), tol_dual=float(td), seed=int(seed),
                   fixed_iterations=bool(fixed))
res = engine.solve(prob, cfg)
print(tag, res.status, res.iterations, np.abs(res.x - g[f"{tag}_x"][res.iterations - 1]).max())
