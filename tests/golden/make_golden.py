"""Generate golden fixtures by running the UNMODIFIED reference (racml).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports racml from /root/reference/pkg/src, observes per-sweep state by
wrapping module attributes (no reference source is edited or copied), and
writes small .npz fixtures next to this script.  The fixtures travel to the
GPU box; /root/reference does not.

Observation points:
  * fit:   racml.elastic_net._col_block (block indices in visit order) and
           racml.elastic_net.z_update (beta_k, xi_{k-1} -> z_k);
  * train: racml.svm.assemble_kernel_block (block indices) and
           racml.svm.solve_block (new block duals);
  * solve: racml.engine.run_sweep (block order) and the sweep_hook (x, y).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import racml  # noqa: E402
import racml.elastic_net as ren  # noqa: E402
import racml.engine as reng  # noqa: E402
import racml.problems as rprob  # noqa: E402
import racml.svm as rsvm  # noqa: E402

from paper_1907_01995_b200 import configs  # noqa: E402


def _save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


# ---------------------------------------------------------------------------
def gen_chunks():
    out = {}
    cases = [(10, 3, 0), (17, 5, 1), (64, 64, 2), (101, 10, 3), (500, 50, 0), (2000, 100, 0)]
    for n, s, seed in cases:
        perm = np.random.default_rng(seed).permutation(n)
        groups = rprob.chunk_indices(perm, s)
        flat = np.concatenate([np.asarray(g, dtype=np.int64) for g in groups])
        lens = np.asarray([len(g) for g in groups], dtype=np.int64)
        out[f"perm_{n}_{s}_{seed}"] = perm.astype(np.int64)
        out[f"flat_{n}_{s}_{seed}"] = flat
        out[f"lens_{n}_{s}_{seed}"] = lens
    # BASELINE config sizes: first two RAC sweeps with seed 0, hashed
    for n, s in [(500, 50), (2000, 100), (5000, 200), (20000, 100), (100000, 500)]:
        rng = np.random.default_rng(0)
        for k in range(2):
            perm = rng.permutation(n)
            groups = rprob.chunk_indices(perm, s)
            flat = np.concatenate([np.asarray(g, dtype=np.int64) for g in groups])
            out[f"sha_{n}_{s}_{k}"] = np.frombuffer(
                hashlib.sha256(flat.tobytes()).digest(), dtype=np.uint8)
    _save("chunks", **out)


# ---------------------------------------------------------------------------
class EnCapture:
    """Per-sweep (blocks, beta, z, xi) of racml.elastic_net.fit."""

    def __init__(self):
        self.blocks, self.cur = [], []
        self.beta, self.z, self.xi = [], [], []

    def __enter__(self):
        self._cb, self._zu = ren._col_block, ren.z_update
        cap = self

        def col_block(X, block):
            cap.cur.append(np.asarray(block, dtype=np.int64).copy())
            return cap._cb(X, block)

        def z_update(beta, xi, gamma, lam, alpha):
            z = cap._zu(beta, xi, gamma, lam, alpha)
            cap.blocks.append(cap.cur)
            cap.cur = []
            cap.beta.append(np.array(beta, dtype=float))
            cap.z.append(np.array(z, dtype=float))
            cap.xi.append(np.asarray(xi, dtype=float) - gamma * (np.asarray(beta) - z))
            return z

        ren._col_block, ren.z_update = col_block, z_update
        return self

    def __exit__(self, *exc):
        ren._col_block, ren.z_update = self._cb, self._zu


def _en_case(tag, X, y, spec, keep_full=None, out=None, block_sweeps=3, save_xy=True):
    with EnCapture() as cap:
        model = ren.fit(X, y, spec)
    K = len(cap.beta)
    keep = range(1, K + 1) if keep_full is None else [k for k in keep_full if k <= K]
    d = out if out is not None else {}
    if save_xy:
        d[f"{tag}_X"] = X
        d[f"{tag}_y"] = y
    d[f"{tag}_params"] = np.array([spec.lam, spec.alpha,
                                   np.nan if spec.gamma is None else spec.gamma,
                                   spec.block_size, spec.iters, spec.seed,
                                   np.nan if spec.tol is None else spec.tol])
    d[f"{tag}_mode"] = np.array(rprob.Mode(spec.mode).value)
    d[f"{tag}_sweeps_kept"] = np.asarray(list(keep), dtype=np.int64)
    for k in keep:
        d[f"{tag}_beta_{k}"] = cap.beta[k - 1]
        d[f"{tag}_z_{k}"] = cap.z[k - 1]
        d[f"{tag}_xi_{k}"] = cap.xi[k - 1]
    for k in range(1, min(K, block_sweeps) + 1):
        d[f"{tag}_blocks_{k}"] = np.concatenate(cap.blocks[k - 1])
        d[f"{tag}_blocklens_{k}"] = np.asarray([b.size for b in cap.blocks[k - 1]])
    d[f"{tag}_norms"] = np.asarray([[np.linalg.norm(b), np.linalg.norm(z), np.linalg.norm(x)]
                                    for b, z, x in zip(cap.beta, cap.z, cap.xi)])
    d[f"{tag}_final_beta"] = model.beta
    d[f"{tag}_final_z"] = model.z
    d[f"{tag}_final_xi"] = model.xi
    d[f"{tag}_final"] = np.array([model.gamma, model.iterations, model.residual,
                                  ren.objective(X, y, model.beta, spec.lam, spec.alpha),
                                  ren.objective(X, y, model.z, spec.lam, spec.alpha)])
    return d


def gen_en():
    Mode = rprob.Mode
    d = {}
    rng = np.random.default_rng(101)
    X = rng.standard_normal((60, 40))
    y = X @ (rng.standard_normal(40) * (rng.random(40) < 0.3)) + 0.1 * rng.standard_normal(60)
    _en_case("lasso_rac", X, y, ren.ElasticNetSpec(lam=0.1, alpha=1.0, gamma=None,
                                                   block_size=7, iters=25, seed=3), out=d)
    rng = np.random.default_rng(102)
    X = rng.standard_normal((50, 30))
    y = rng.standard_normal(50)
    _en_case("ridge_rp", X, y, ren.ElasticNetSpec(lam=0.5, alpha=0.0, gamma=1.0, block_size=8,
                                                  iters=25, mode=Mode.RP, seed=5), out=d)
    rng = np.random.default_rng(103)
    X = rng.standard_normal((80, 24))
    y = X @ rng.standard_normal(24) + 0.3 * rng.standard_normal(80)
    _en_case("enet_tol", X, y, ren.ElasticNetSpec(lam=0.05, alpha=0.5, gamma=0.3, block_size=6,
                                                  iters=5000, seed=1, tol=1e-8),
             keep_full=[1, 2, 3, 10], out=d)
    # lam = 0: plain least squares, gamma auto -> 1 (elastic_net.py:95-96)
    rng = np.random.default_rng(104)
    X = rng.standard_normal((40, 12))
    y = rng.standard_normal(40)
    _en_case("ls_lam0", X, y, ren.ElasticNetSpec(lam=0.0, alpha=1.0, block_size=5, iters=15,
                                                 seed=2), out=d)
    # block_size > n is clamped (elastic_net.py:175)
    rng = np.random.default_rng(105)
    X = rng.standard_normal((20, 6))
    y = rng.standard_normal(20)
    _en_case("clamp_bs", X, y, ren.ElasticNetSpec(lam=0.2, alpha=0.7, gamma=0.5, block_size=50,
                                                  iters=6, seed=0), out=d)
    _save("en_small", **d)

    c1 = configs.config1()
    spec = ren.ElasticNetSpec(lam=c1.lam, alpha=c1.alpha, gamma=c1.gamma,
                              block_size=c1.block_size, iters=c1.iters, seed=c1.seed)
    d = _en_case("cfg1", c1.X, c1.y, spec, keep_full=[1, 2, 5, 10, 25, 50])
    del d["cfg1_X"], d["cfg1_y"]   # regenerated from the seed on the GPU box
    _save("en_config1", **d)

    c2 = configs.config2(scale=0.1)
    spec = ren.ElasticNetSpec(lam=c2.lam, alpha=c2.alpha, gamma=c2.gamma,
                              block_size=c2.block_size, iters=c2.iters, seed=c2.seed, tol=c2.tol)
    d = _en_case("cfg2s", c2.X, c2.y, spec, keep_full=[1, 2, 5, 10])
    del d["cfg2s_X"], d["cfg2s_y"]
    _save("en_config2_small", **d)


# ---------------------------------------------------------------------------
class SvmCapture:
    def __init__(self):
        self.block_idx, self.block_z = [], []

    def __enter__(self):
        self._akb, self._sb = rsvm.assemble_kernel_block, rsvm.solve_block
        cap = self

        def akb(X, y, block, kernel, cache=None, with_strip=False):
            cap.block_idx.append(np.asarray(block, dtype=np.int64).copy())
            return cap._akb(X, y, block, kernel, cache=cache, with_strip=with_strip)

        def sb(system, chol=None):
            out = cap._sb(system, chol)
            cap.block_z.append(np.array(out, dtype=float))
            return out

        rsvm.assemble_kernel_block, rsvm.solve_block = akb, sb
        return self

    def __exit__(self, *exc):
        rsvm.assemble_kernel_block, rsvm.solve_block = self._akb, self._sb


def _svm_case(tag, X, y, C, kernel, cfg, out, keep=None, save_xy=True):
    with SvmCapture() as cap:
        model, diag = rsvm.train(X, y, C, kernel, cfg, return_diagnostics=True)
    n = X.shape[0]
    p = len(rprob.chunk_indices(np.arange(n), cfg.block_size))
    z = np.zeros(n)
    t = 0.0
    nu = 0.0
    zs, nus = [], []
    for k in range(diag.iterations):
        for b in range(p):
            idx = cap.block_idx[k * p + b]
            nz = cap.block_z[k * p + b]
            t += float(y[idx] @ (nz - z[idx]))
            z[idx] = nz
        nu -= cfg.beta_penalty * t
        zs.append(z.copy())
        nus.append(nu)
    assert np.array_equal(z, diag.duals) and nu == diag.eq_dual
    if save_xy:
        out[f"{tag}_X"] = X
        out[f"{tag}_y"] = y
    out[f"{tag}_params"] = np.array([C, cfg.block_size, cfg.beta_penalty, cfg.max_iters,
                                     cfg.tol_primal, cfg.tol_dual, cfg.seed,
                                     float(cfg.fixed_iterations), kernel.sigma])
    out[f"{tag}_kernel"] = np.array(kernel.kind)
    out[f"{tag}_mode"] = np.array(rprob.Mode(cfg.mode).value)
    if keep is None:
        out[f"{tag}_z"] = np.asarray(zs)
    else:
        kept = [k for k in keep if k <= len(zs)]
        out[f"{tag}_sweeps_kept"] = np.asarray(kept, dtype=np.int64)
        for k in kept:
            out[f"{tag}_z_{k}"] = zs[k - 1]
        out[f"{tag}_znorms"] = np.asarray([np.linalg.norm(v) for v in zs])
        if kernel.kind == "linear":
            w = X.T @ (y * z)        # linear kernel: z'Qz = ||X'(y*z)||^2 (test_svm.py:173)
            out[f"{tag}_dual_objective"] = np.array(0.5 * float(w @ w) - float(z.sum()))
    out[f"{tag}_nu"] = np.asarray(nus)
    out[f"{tag}_primal"] = diag.primal_residual_history
    out[f"{tag}_dual"] = diag.dual_residual_history
    out[f"{tag}_iterations"] = np.array(diag.iterations)
    out[f"{tag}_status"] = np.array(rprob.Status(diag.status).value)
    out[f"{tag}_bias"] = np.array(model.bias)
    out[f"{tag}_blocks_1"] = np.concatenate(cap.block_idx[:p])


def gen_svm():
    Mode, SolverConfig = rprob.Mode, rprob.SolverConfig
    d = {}
    rng = np.random.default_rng(201)
    n = 120
    y = np.where(np.arange(n) < n // 2, 1.0, -1.0)
    X = rng.standard_normal((n, 5)) + y[:, None] * 0.6
    y[rng.choice(n, 6, replace=False)] *= -1
    _svm_case("lin", X, y, 1.0, rsvm.KernelSpec("linear"),
              SolverConfig(mode=Mode.RAC, block_size=16, beta_penalty=1.0, max_iters=25,
                           tol_primal=1e-6, tol_dual=1e-6, seed=0), d)
    rng = np.random.default_rng(202)
    n = 90
    y = np.where(np.arange(n) < n // 2, 1.0, -1.0)
    X = rng.standard_normal((n, 3)) + y[:, None] * 0.8
    _svm_case("gauss", X, y, 0.5, rsvm.KernelSpec("gaussian", 1.3),
              SolverConfig(mode=Mode.RAC, block_size=10, beta_penalty=0.9, max_iters=30,
                           tol_primal=1e-6, tol_dual=1e-6, seed=4), d)
    _svm_case("gauss_rp", X, y, 0.5, rsvm.KernelSpec("gaussian", 1.3),
              SolverConfig(mode=Mode.RP, block_size=10, beta_penalty=0.9, max_iters=20,
                           tol_primal=1e-6, tol_dual=1e-6, seed=4), d)
    c4 = configs.config4(scale=0.05)
    _svm_case("cfg4s", c4.X, c4.labels, c4.C, rsvm.KernelSpec("linear"),
              SolverConfig(mode=Mode.RAC, block_size=c4.block_size, beta_penalty=c4.beta,
                           max_iters=20, tol_primal=1e-6, tol_dual=1e-6, seed=0), d)
    _save("svm_small", **d)


# ---------------------------------------------------------------------------
def _qp_case(tag, prob, cfg, out):
    orders, xs, ys = [], [], []
    orig = reng.run_sweep

    def rs(problem, x, y, order, beta, chol_cache=None, piece_cache=None):
        orders.append(np.concatenate([np.asarray(g, dtype=np.int64) for g in order]))
        return orig(problem, x, y, order, beta, chol_cache=chol_cache, piece_cache=piece_cache)

    reng.run_sweep = rs
    try:
        res = reng.solve(prob, cfg, sweep_hook=lambda k, x, y: (xs.append(x.copy()),
                                                                 ys.append(y.copy())))
    finally:
        reng.run_sweep = orig
    for name, v in (("c", prob.c), ("H", prob.H), ("A", prob.A), ("b", prob.b),
                    ("lower", prob.lower), ("upper", prob.upper)):
        if v is not None:
            out[f"{tag}_{name}"] = np.asarray(v, dtype=float)
    out[f"{tag}_params"] = np.array([cfg.block_size, cfg.beta_penalty, cfg.max_iters,
                                     cfg.tol_primal, cfg.tol_dual, cfg.seed,
                                     float(cfg.fixed_iterations)])
    out[f"{tag}_mode"] = np.array(rprob.Mode(cfg.mode).value)
    out[f"{tag}_x"] = np.asarray(xs)
    out[f"{tag}_y"] = np.asarray(ys) if ys and ys[0].size else np.zeros((len(xs), 0))
    out[f"{tag}_order_1"] = orders[0]
    out[f"{tag}_primal"] = res.primal_residual_history
    out[f"{tag}_primal_l1"] = res.primal_l1_history
    out[f"{tag}_dual"] = res.dual_residual_history
    out[f"{tag}_iterations"] = np.array(res.iterations)
    out[f"{tag}_status"] = np.array(rprob.Status(res.status).value)


def _rand_qp(seed, n, m, bounded):
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n)) / np.sqrt(n)
    H = G @ G.T + 0.5 * np.eye(n)
    H = 0.5 * (H + H.T)
    A = rng.standard_normal((m, n))
    c = rng.standard_normal(n)
    kw = {}
    if bounded:
        kw = dict(lower=np.full(n, -0.3), upper=np.full(n, 0.3))
        xf = rng.uniform(-0.25, 0.25, size=n)
    else:
        xf = rng.standard_normal(n)
    return rprob.QpProblem(c=c, H=H, A=A, b=A @ xf, **kw)


def gen_qp():
    Mode, SolverConfig = rprob.Mode, rprob.SolverConfig
    d = {}
    _qp_case("box_rac", _rand_qp(301, 30, 4, True),
             SolverConfig(mode=Mode.RAC, block_size=7, beta_penalty=1.0, max_iters=40,
                          tol_primal=1e-9, tol_dual=1e-9, seed=2), d)
    _qp_case("box_rp", _rand_qp(302, 24, 3, True),
             SolverConfig(mode=Mode.RP, block_size=6, beta_penalty=0.8, max_iters=40,
                          tol_primal=1e-9, tol_dual=1e-9, seed=3), d)
    _qp_case("free_cyclic", _rand_qp(303, 20, 5, False),
             SolverConfig(mode=Mode.CYCLIC, block_size=5, beta_penalty=1.0, max_iters=40,
                          tol_primal=1e-12, tol_dual=1e-12, seed=0, fixed_iterations=True), d)
    _qp_case("medium_box", _rand_qp(304, 300, 40, True),
             SolverConfig(mode=Mode.RAC, block_size=50, beta_penalty=1.0, max_iters=60,
                          tol_primal=1e-7, tol_dual=1e-7, seed=1), d)
    # no equality constraints, H only, one-sided bounds
    rng = np.random.default_rng(305)
    G = rng.standard_normal((16, 16))
    H = G @ G.T / 16 + 0.2 * np.eye(16)
    H = 0.5 * (H + H.T)
    lo = np.where(rng.random(16) < 0.5, -0.2, -np.inf)
    hi = np.where(rng.random(16) < 0.5, 0.2, np.inf)
    _qp_case("h_only", rprob.QpProblem(c=rng.standard_normal(16), H=H, lower=lo, upper=hi),
             SolverConfig(mode=Mode.RAC, block_size=4, beta_penalty=1.0, max_iters=30,
                          tol_primal=1e-10, tol_dual=1e-10, seed=7), d)
    # divergent 3-block cyclic counterexample (test_engine.py:326-340)
    A = np.array([[1.0, 1.0, 1.0], [1.0, 1.0, 2.0], [1.0, 2.0, 2.0]])
    _qp_case("diverge", rprob.QpProblem(c=np.array([1.0, -2.0, 0.5]), A=A, b=np.ones(3)),
             SolverConfig(mode=Mode.CYCLIC, block_size=1, beta_penalty=1.0, max_iters=1500,
                          tol_primal=1e-12, tol_dual=1e-12, seed=0), d)
    _save("qp_small", **d)


# ---------------------------------------------------------------------------
def gen_block_and_prox():
    d = {}
    rng = np.random.default_rng(401)
    for i in range(16):
        s = int(rng.integers(3, 24))
        G = rng.standard_normal((s, s))
        M = G @ G.T + 0.3 * np.eye(s)
        r = rng.standard_normal(s) * 3
        lo = -rng.random(s)
        hi = rng.random(s)
        if i % 4 == 3:
            lo[rng.random(s) < 0.3] = -np.inf
            hi[rng.random(s) < 0.3] = np.inf
        x = reng.solve_block(reng.BlockSystem(M, r, lo, hi))
        d[f"blk{i}_M"], d[f"blk{i}_r"], d[f"blk{i}_lo"], d[f"blk{i}_hi"], d[f"blk{i}_x"] = \
            M, r, lo, hi, x
    d["blk_count"] = np.array(16)
    a = rng.standard_normal(2000) * 3
    b = rng.random(2000)
    beta = rng.standard_normal(2000) * 3
    xi = rng.standard_normal(2000) * 3
    d["prox_a"], d["prox_b"] = a, b
    d["prox_st"] = np.asarray([ren.soft_threshold(float(ai), float(bi)) for ai, bi in zip(a, b)])
    d["prox_beta"], d["prox_xi"] = beta, xi
    d["prox_z"] = ren.z_update(beta, xi, 0.7, 0.4, 0.3)
    _save("block_prox", **d)


# ---------------------------------------------------------------------------
def gen_sparse():
    """racml fit on scipy CSC designs (the test_elastic_net.py:261-269 recipe and a larger,
    1%-dense one): per-sweep iterates of the reference's sparse column-block path."""
    import scipy.sparse as sps
    d = {}
    rng = np.random.default_rng(15)
    X = sps.csc_matrix(np.where(rng.random((30, 40)) < 0.2, rng.standard_normal((30, 40)), 0.0))
    y = rng.standard_normal(30)
    _en_case("ref", X, y, ren.ElasticNetSpec(lam=0.05, alpha=1.0, block_size=16, iters=50, seed=7),
             keep_full=[1, 2, 5, 10, 25, 50], out=d, save_xy=False)
    d["ref_X"] = X.toarray()
    d["ref_y"] = y
    rng = np.random.default_rng(16)
    X = sps.random(1500, 2400, density=0.01, format="csc", random_state=np.random.RandomState(16),
                   data_rvs=lambda k: rng.standard_normal(k))
    y = X @ (rng.standard_normal(2400) * (rng.random(2400) < 0.05)) + 0.01 * rng.standard_normal(1500)
    _en_case("big", X, y, ren.ElasticNetSpec(lam=0.02, alpha=0.9, gamma=None, block_size=120, iters=30, seed=2),
             keep_full=[1, 2, 5, 10, 30], out=d, save_xy=False)
    d["big_data"], d["big_indices"], d["big_indptr"] = X.data, X.indices, X.indptr
    d["big_shape"] = np.array(X.shape)
    d["big_y"] = y
    _save("en_sparse", **d)


# ---------------------------------------------------------------------------
def gen_consensus():
    """racml.elastic_net.consensus_fit on direct-route (p <= n_i), Woodbury-route (p > n_i)
    and mixed group shapes, with and without a tolerance."""
    d = {}
    cases = [
        ("direct", 400, 12, dict(lam=0.1, alpha=0.7, gamma=0.5, block_size=4, iters=40, seed=3)),
        ("woodbury", 40, 90, dict(lam=0.05, alpha=1.0, gamma=1.0, block_size=10, iters=60, seed=4)),
        ("mixed_tol", 61, 20, dict(lam=0.2, alpha=0.5, gamma=None, block_size=7, iters=5000, seed=5, tol=1e-8)),
        ("ridge", 120, 30, dict(lam=0.3, alpha=0.0, gamma=0.8, block_size=6, iters=25, seed=6)),
    ]
    for i, (tag, n, p, kw) in enumerate(cases):
        rng = np.random.default_rng(500 + i)
        X = rng.standard_normal((n, p))
        y = X @ (rng.standard_normal(p) * (rng.random(p) < 0.3)) + 0.1 * rng.standard_normal(n)
        spec = ren.ElasticNetSpec(**kw)
        m = ren.consensus_fit(X, y, spec)
        d[f"{tag}_X"], d[f"{tag}_y"] = X, y
        d[f"{tag}_params"] = np.array([spec.lam, spec.alpha, np.nan if spec.gamma is None else spec.gamma,
                                       spec.block_size, spec.iters, spec.seed, np.nan if spec.tol is None else spec.tol])
        d[f"{tag}_beta"], d[f"{tag}_z"], d[f"{tag}_xi"] = m.beta, m.z, m.xi
        d[f"{tag}_final"] = np.array([m.gamma, m.iterations, m.residual])
    _save("consensus", **d)


# ---------------------------------------------------------------------------
# Full BASELINE sizes (VERDICT r01 "next round" #1): the unmodified racml at the
# §8(d) seed-0 recipe.  Inputs are NOT stored (regenerated from the seed on the
# GPU box by paper_1907_01995_b200.configs); kept: iterates at sweeps 1, 2, 5, 10,
# 25, 50, the norms of every sweep, the first sweep's block list, the final
# iterates, objective and iteration count.
FULL_KEEP = [1, 2, 5, 10, 25, 50]


def gen_full_en(cfg: int, iters: int | None = None):
    import time
    c = configs.GENERATORS[cfg]()
    spec = ren.ElasticNetSpec(lam=c.lam, alpha=c.alpha, gamma=c.gamma, block_size=c.block_size,
                              iters=iters or c.iters, seed=c.seed, tol=c.tol)
    t0 = time.perf_counter()
    d = _en_case(f"cfg{cfg}", c.X, c.y, spec, keep_full=FULL_KEEP, block_sweeps=1, save_xy=False)
    d[f"cfg{cfg}_blocks_1"] = d[f"cfg{cfg}_blocks_1"].astype(np.int32)
    d[f"cfg{cfg}_seconds"] = np.array(time.perf_counter() - t0)
    print(f"config {cfg}: {int(d[f'cfg{cfg}_final'][1])} sweeps in {float(d[f'cfg{cfg}_seconds']):.1f} s")
    _save(f"en_config{cfg}_full", **d)


def gen_full_svm(sweeps: int = 50):
    import time
    Mode, SolverConfig = rprob.Mode, rprob.SolverConfig
    c = configs.config4()
    d = {}
    t0 = time.perf_counter()
    _svm_case("cfg4", c.X, c.labels, c.C, rsvm.KernelSpec("linear"),
              SolverConfig(mode=Mode.RAC, block_size=c.block_size, beta_penalty=c.beta,
                           max_iters=sweeps, tol_primal=c.tol_primal, tol_dual=c.tol_dual, seed=0),
              d, keep=FULL_KEEP, save_xy=False)
    d["cfg4_blocks_1"] = d["cfg4_blocks_1"].astype(np.int32)
    d["cfg4_seconds"] = np.array(time.perf_counter() - t0)
    print(f"config 4: {sweeps} sweeps in {float(d['cfg4_seconds']):.1f} s")
    _save("svm_config4_full", **d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["chunks", "en", "svm", "qp", "block"]
    if "consensus" in which:
        gen_consensus()
    if "sparse" in which:
        gen_sparse()
    if "full2" in which:
        gen_full_en(2)
    if "full3" in which:
        gen_full_en(3)
    if "full5" in which:
        gen_full_en(5, iters=50)
    if "full4" in which:
        gen_full_svm(50)
    if "chunks" in which:
        gen_chunks()
    if "block" in which:
        gen_block_and_prox()
    if "qp" in which:
        gen_qp()
    if "svm" in which:
        gen_svm()
    if "en" in which:
        gen_en()
    print("racml", racml.__version__)
