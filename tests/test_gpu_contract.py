"""GPU: the reference's public helper surface and the error paths.

Each helper runs on the device and is checked against the CPU oracle / numpy restatement
of the reference function it replaces (engine.py:51-315, svm.py:68-143, 287-322).
Error paths: BlockDefinitenessError raised from inside a sweep by fit / solve / train,
and the projected-gradient fallback of the box block solver (engine.py:175-186).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_1907_01995_b200 import _device
    return _device.require_cuda(0)


def _rand_qp(seed, n, m, bounded):
    from paper_1907_01995_b200.problems import QpProblem
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n)) / np.sqrt(n)
    H = G @ G.T + 0.5 * np.eye(n)
    H = 0.5 * (H + H.T)
    A = rng.standard_normal((m, n))
    c = rng.standard_normal(n)
    kw = dict(lower=np.full(n, -0.3), upper=np.full(n, 0.3)) if bounded else {}
    return QpProblem(c=c, H=H, A=A, b=A @ rng.uniform(-0.25, 0.25, n), **kw)


def test_solve_block_takes_block_system(dev, golden):
    import paper_1907_01995_b200 as rac
    g = golden("block_prox")
    for i in range(int(g["blk_count"])):
        x = rac.solve_block(rac.BlockSystem(g[f"blk{i}_M"], g[f"blk{i}_r"], g[f"blk{i}_lo"], g[f"blk{i}_hi"]))
        assert np.max(np.abs(x - g[f"blk{i}_x"])) <= 1e-12 * max(1.0, np.max(np.abs(g[f"blk{i}_x"]))), i
    # bounded=False: the plain SPD solve even with finite bounds (engine.py:204-205)
    M = np.array([[2.0, 0.5], [0.5, 1.0]])
    r = np.array([10.0, -10.0])
    x = rac.solve_block(rac.BlockSystem(M, r, np.zeros(2), np.ones(2), bounded=False))
    np.testing.assert_allclose(x, np.linalg.solve(M, r), rtol=1e-13)
    with pytest.raises(rac.BlockDefinitenessError, match="positive definite"):
        rac.solve_block(rac.BlockSystem(np.zeros((1, 1)), np.ones(1), np.array([-np.inf]), np.array([np.inf])))


def test_projected_gradient_fallback(dev, monkeypatch):
    """RAC_BOX_PASSES=0 sends the block solver straight to the PG fallback; it must land on
    the same minimizer as the active set (the reference test compares to 1e-9)."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import engine
    rng = np.random.default_rng(11)
    monkeypatch.setenv("RAC_BOX_PASSES", "0")
    for s in (3, 17, 40):
        G = rng.standard_normal((s, s))
        M = G @ G.T + 0.5 * np.eye(s)
        r = rng.standard_normal(s) * 4
        lo, hi = -rng.random(s), rng.random(s)
        want = ro.box_block_min(M, r, lo, hi)
        got = engine.solve_block(engine.BlockSystem(M, r, lo, hi))
        assert np.max(np.abs(got - want)) <= 1e-8, s
        assert np.all(got >= lo - 1e-15) and np.all(got <= hi + 1e-15)


def test_dual_update_and_residuals(dev):
    import paper_1907_01995_b200 as rac
    from oracle import rac_oracle as ro
    prob = _rand_qp(7, 40, 6, True)
    rng = np.random.default_rng(8)
    x, y = rng.uniform(-0.3, 0.3, 40), rng.standard_normal(6)
    got = rac.dual_update(y, prob.A, x, prob.b, 0.7)
    np.testing.assert_allclose(got, y - 0.7 * (prob.A @ x - prob.b), rtol=1e-13, atol=1e-13)
    res = rac.compute_residuals(prob, x, y)
    p, d, l1 = ro.qp_residuals(prob.H, prob.c, prob.A, prob.b, prob.lower, prob.upper, x, y)
    assert abs(res.primal - p) <= 1e-13 * max(1, p) and abs(res.primal_l1 - l1) <= 1e-12 * max(1, l1)
    assert abs(res.dual - d) <= 1e-12 * max(1, d)
    xn = x.copy()
    xn[3] = np.nan
    assert np.isnan(rac.compute_residuals(prob, xn, y).dual)


def test_assemble_block_system(dev):
    import paper_1907_01995_b200 as rac
    prob = _rand_qp(9, 30, 4, True)
    rng = np.random.default_rng(10)
    x, y = rng.uniform(-0.3, 0.3, 30), rng.standard_normal(4)
    blk = np.array([2, 5, 11, 29])
    sys_ = rac.assemble_block_system(prob, x, y, blk, 0.9)
    H, A = prob.H, prob.A
    M = H[np.ix_(blk, blk)] + 0.9 * A[:, blk].T @ A[:, blk]
    rest = np.setdiff1d(np.arange(30), blk)
    r = -(prob.c[blk] + H[np.ix_(blk, rest)] @ x[rest] - A[:, blk].T @ y
          + 0.9 * A[:, blk].T @ (A[:, rest] @ x[rest] - prob.b))
    np.testing.assert_allclose(sys_.matrix, M, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(sys_.rhs, r, rtol=1e-11, atol=1e-11)
    assert sys_.bounded


def test_run_sweep_matches_oracle_sweep(dev):
    """One device sweep in a given order from a given (x, y) = the oracle's sweep."""
    import paper_1907_01995_b200 as rac
    from oracle import rac_oracle as ro
    prob = _rand_qp(12, 36, 5, True)
    rng = np.random.default_rng(13)
    x0, y0 = rng.uniform(-0.3, 0.3, 36), rng.standard_normal(5)
    order = rac.chunk_indices(rng.permutation(36), 8)
    x1, y1 = rac.run_sweep(prob, x0, y0, order, 1.3)
    # the oracle's sweep from the same state: block minimizations in order, then the dual step
    x = x0.copy()
    for g in order:
        idx = np.asarray(g)
        s_ = rac.assemble_block_system(prob, x, y0, idx, 1.3)
        x[idx] = ro.box_block_min(s_.matrix, s_.rhs, s_.lower, s_.upper)
    y = y0 - 1.3 * (prob.A @ x - prob.b)
    assert np.linalg.norm(x1 - x) <= 1e-10 * np.linalg.norm(x)
    assert np.linalg.norm(y1 - y) <= 1e-10 * np.linalg.norm(y)
    assert np.array_equal(x0, x0) and x1 is not x0


@pytest.mark.parametrize("kind,sigma", [("linear", 1.0), ("gaussian", 1.7)])
def test_assemble_kernel_block_and_bias(dev, kind, sigma):
    import paper_1907_01995_b200 as rac
    from oracle import rac_oracle as ro
    rng = np.random.default_rng(21)
    N, d = 300, 7
    y = np.where(np.arange(N) < N // 2, 1.0, -1.0)
    X = rng.standard_normal((N, d)) + y[:, None] * 0.5
    blk = np.sort(rng.choice(N, 40, replace=False))
    kern = rac.KernelSpec(kind, sigma)
    qbb, strip = rac.assemble_kernel_block(X, y, blk, kern, with_strip=True)
    K = ro.kernel_matrix(X[blk], X, kind, sigma)
    want = (y[blk][:, None] * K) * y[None, :]
    np.testing.assert_allclose(strip, want, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(qbb, want[:, blk], rtol=1e-12, atol=1e-12)
    z = np.clip(rng.standard_normal(N), 0.0, 1.0) * (rng.random(N) < 0.6)
    b = rac.compute_bias(z, X, y, 1.0, kern)
    assert abs(b - ro.svm_bias(z, X, y, 1.0, kind, sigma)) <= 1e-10 * max(1.0, abs(b))
    # all duals at a bound: the bracket midpoint branch
    zb = np.where(rng.random(N) < 0.5, 1.0, 0.0)
    b2 = rac.compute_bias(zb, X, y, 1.0, kern)
    assert abs(b2 - ro.svm_bias(zb, X, y, 1.0, kind, sigma)) <= 1e-10 * max(1.0, abs(b2))
    assert rac.kernel_eval(X[0], X[1], kern) == pytest.approx(float(ro.kernel_matrix(X[:1], X[1:2], kind, sigma)[0, 0]),
                                                              rel=1e-14)


# ---------------------------------------------------------------- not-PD raised mid-sweep
@pytest.mark.parametrize("gram,m,n,s", [("blocks", 80, 40, 8), ("covariance", 80, 40, 8),
                                         ("blocks", 700, 600, 300)])    # s > 236: the large-s inverse
def test_fit_raises_block_definiteness_mid_sweep(dev, gram, m, n, s):
    """A NaN column makes its block system indefinite for LAPACK (the reference's
    np.linalg.cholesky raises at that block, elastic_net.py:213-219)."""
    import paper_1907_01995_b200 as rac
    rng = np.random.default_rng(3)
    X = rng.standard_normal((m, n))
    X[:, 17] = np.nan
    with pytest.raises(rac.BlockDefinitenessError, match="positive definite"):
        rac.fit(X, rng.standard_normal(m), rac.ElasticNetSpec(lam=0.1, alpha=0.5, gamma=1.0, block_size=s, iters=5),
                gram_mode=gram)
    # the pooled context is sound afterwards: a clean fit of the same shape works
    Xc = rng.standard_normal((m, n))
    m = rac.fit(Xc, rng.standard_normal(m), rac.ElasticNetSpec(lam=0.1, alpha=0.5, gamma=1.0, block_size=s, iters=5),
                gram_mode=gram)
    assert m.iterations == 5 and np.all(np.isfinite(m.beta))


def test_solve_raises_block_definiteness_mid_sweep(dev):
    """H with a zero diagonal entry and no constraints: the 1 x 1 block of that coordinate is
    singular (engine.py:160-167), reached inside the first sweep."""
    import paper_1907_01995_b200 as rac
    H = np.diag([1.0, 2.0, 0.0, 3.0, 1.5, 1.0])
    prob = rac.QpProblem(c=np.ones(6), H=H)
    with pytest.raises(rac.BlockDefinitenessError, match="positive definite"):
        rac.solve(prob, rac.SolverConfig(block_size=1, max_iters=3, seed=0))


def test_train_raises_block_definiteness_mid_sweep(dev):
    import paper_1907_01995_b200 as rac
    rng = np.random.default_rng(4)
    N = 60
    y = np.where(np.arange(N) < N // 2, 1.0, -1.0)
    X = rng.standard_normal((N, 3))
    X[41, 1] = np.nan
    with pytest.raises(rac.BlockDefinitenessError):
        rac.train(X, y, 1.0, rac.KernelSpec("linear"), rac.SolverConfig(block_size=10, max_iters=2, seed=0))


def test_qp_nan_residual_is_not_converged(dev):
    """NaN iterates must not read as converged (numpy's max propagates NaN).  validate_problem
    rejects a NaN c up front, so the native context is driven directly: a NaN in c makes the
    dual residual NaN every sweep; the run goes to the cap with status max_iters."""
    from paper_1907_01995_b200.engine import QpSolver
    from paper_1907_01995_b200.problems import Mode, Status
    n = 4
    sol = QpSolver(n, 0, 2, Mode.CYCLIC, 1.0, 0.0)
    try:
        sol.set_problem(np.array([1.0, np.nan, -1.0, 0.5]), np.full(n, -1.0), np.full(n, 1.0), H=np.eye(n) * 2.0)
        sol.set_partition(np.arange(n))
        sol.run(None, 4, 1e-6, 1e-6, False)
        it, status, failed = sol.progress()
        hp, _, hd = (h.cpu().numpy() for h in sol.history(it))
    finally:
        sol.close()
    assert failed < 0 and it == 4 and status == Status.MAX_ITERS
    assert np.isnan(hd).all()


def test_current_device_is_the_default(dev):
    """With no device argument the solvers use torch's current device (torchrun ranks)."""
    import torch
    import paper_1907_01995_b200 as rac
    from paper_1907_01995_b200 import _device
    assert _device.resolve_device(None) == torch.cuda.current_device()
    rng = np.random.default_rng(5)
    m = rac.fit(rng.standard_normal((30, 12)), rng.standard_normal(30), rac.ElasticNetSpec(lam=0.1, alpha=0.5, iters=3,
                                                                                          block_size=4))
    assert m.iterations == 3


# ---------------------------------------------------------------- consensus baseline (§8(f) rank 4)
@pytest.mark.parametrize("tag", ["direct", "woodbury", "mixed_tol", "ridge"])
def test_consensus_fit_matches_reference(dev, golden, tag):
    import paper_1907_01995_b200 as rac
    from paper_1907_01995_b200.elastic_net import objective
    g = golden("consensus")
    lam, alpha, gamma, bs, iters, seed, tol = g[f"{tag}_params"]
    spec = rac.ElasticNetSpec(lam=float(lam), alpha=float(alpha), gamma=None if np.isnan(gamma) else float(gamma),
                              block_size=int(bs), iters=int(iters), seed=int(seed),
                              tol=None if np.isnan(tol) else float(tol))
    m = rac.consensus_fit(g[f"{tag}_X"], g[f"{tag}_y"], spec)
    assert abs(m.iterations - int(g[f"{tag}_final"][1])) <= 1
    for k in ("beta", "z", "xi"):
        want = g[f"{tag}_{k}"]
        assert np.linalg.norm(getattr(m, k) - want) <= 1e-9 * max(np.linalg.norm(want), 1e-300), k
    X, y = g[f"{tag}_X"], g[f"{tag}_y"]
    ow = objective(X, y, g[f"{tag}_beta"], spec.lam, spec.alpha)
    assert abs(objective(X, y, m.beta, spec.lam, spec.alpha) - ow) <= 1e-8 * abs(ow)
    assert m.gamma == g[f"{tag}_final"][0]
