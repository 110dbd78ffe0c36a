"""GPU parity: dense box-QP engine (engine.solve) and the SVM dual (svm.train)
vs the reference's golden fixtures and the CPU oracle.

Bars: block orders bit-exact; iterates <= 1e-9 relative L2 for the first 50
sweeps; final objective <= 1e-8 relative; same iteration count and status.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-9
OBJ_TOL = 1e-8


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


@pytest.fixture(scope="module")
def dev():
    from paper_1907_01995_b200 import _device
    return _device.require_cuda(0)


# ---------------------------------------------------------------- box block solver
def test_box_block_min_matches_reference(dev, golden):
    from paper_1907_01995_b200 import engine
    g = golden("block_prox")
    for i in range(int(g["blk_count"])):
        x = engine.solve_block(g[f"blk{i}_M"], g[f"blk{i}_r"], g[f"blk{i}_lo"], g[f"blk{i}_hi"])
        assert np.max(np.abs(x - g[f"blk{i}_x"])) <= 1e-12 * max(1.0, np.max(np.abs(g[f"blk{i}_x"]))), i


def test_box_block_min_vs_oracle_random(dev):
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import engine
    rng = np.random.default_rng(5)
    for s in (1, 2, 7, 33, 64, 100, 130):
        G = rng.standard_normal((s, s))
        M = G @ G.T + 0.3 * np.eye(s)
        r = rng.standard_normal(s) * 3
        lo, hi = -rng.random(s), rng.random(s)
        want = ro.box_block_min(M, r, lo, hi)
        got = engine.solve_block(M, r, lo, hi)
        assert np.max(np.abs(got - want)) <= 1e-10 * max(1.0, np.max(np.abs(want))), s


def test_box_block_not_pd_raises(dev):
    from paper_1907_01995_b200 import engine
    with pytest.raises(engine.BlockDefinitenessError, match="positive definite"):
        engine.solve_block(np.zeros((1, 1)), np.ones(1), np.array([-np.inf]), np.array([np.inf]))


# ---------------------------------------------------------------- engine.solve
@pytest.mark.parametrize("tag", ["box_rac", "box_rp", "free_cyclic", "medium_box", "h_only", "diverge"])
def test_solve_matches_reference(dev, golden, tag):
    from paper_1907_01995_b200 import engine
    from paper_1907_01995_b200.problems import Mode, QpProblem, SolverConfig
    g = golden("qp_small")
    bs, beta, iters, tp, td, seed, fixed = g[f"{tag}_params"]
    prob = QpProblem(c=g[f"{tag}_c"], H=g.get(f"{tag}_H"), A=g.get(f"{tag}_A"), b=g.get(f"{tag}_b"),
                     lower=g[f"{tag}_lower"], upper=g[f"{tag}_upper"])
    cfg = SolverConfig(mode=Mode(str(g[f"{tag}_mode"])), block_size=int(bs), beta_penalty=float(beta),
                       max_iters=int(iters), tol_primal=float(tp), tol_dual=float(td), seed=int(seed),
                       fixed_iterations=bool(fixed))
    xs, ys = [], []
    res = engine.solve(prob, cfg, sweep_hook=lambda k, x, y: (xs.append(x), ys.append(y)))
    assert res.status.value == str(g[f"{tag}_status"])
    assert abs(res.iterations - int(g[f"{tag}_iterations"])) <= 1
    for k in range(min(res.iterations, int(g[f"{tag}_iterations"]), 50)):
        assert rel(xs[k], g[f"{tag}_x"][k]) <= ITER_TOL, (tag, k)
        if ys[k].size:
            assert rel(ys[k], g[f"{tag}_y"][k]) <= ITER_TOL, (tag, k)
    n = min(res.iterations, len(g[f"{tag}_primal"]), 50)
    np.testing.assert_allclose(res.primal_residual_history[:n], g[f"{tag}_primal"][:n], rtol=1e-7, atol=1e-13)
    np.testing.assert_allclose(res.dual_residual_history[:n], g[f"{tag}_dual"][:n], rtol=1e-7, atol=1e-13)
    if prob.H is not None and tag != "diverge":
        from oracle import rac_oracle as ro
        want = ro.qp_objective(prob.H, prob.c, g[f"{tag}_x"][res.iterations - 1])
        got = ro.qp_objective(prob.H, prob.c, res.x)
        assert abs(got - want) <= OBJ_TOL * max(abs(want), 1e-12)


@pytest.mark.parametrize("tag", ["box_rac", "medium_box", "h_only"])
def test_solve_two_barriers_per_block(dev, golden, tag, monkeypatch):
    """RAC_QP_LL=0 keeps the chain's two grid barriers per block (the default hands hx at the next
    block's coordinates and the constraint rows' partial to CTA 0 as tagged words and has one):
    same per-sweep iterates against the reference's golden vectors."""
    monkeypatch.setenv("RAC_QP_LL", "0")
    test_solve_matches_reference(dev, golden, tag)


@pytest.mark.parametrize("ll", ["0", "1"])
def test_train_handoff_modes_agree_with_oracle(dev, ll, monkeypatch):
    """svm.train (one constraint row: the tagged hx / partial hand-off path) on a shape with a short
    last block and several column strips, in both hand-off modes, per sweep against the oracle."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import svm
    from paper_1907_01995_b200.problems import SolverConfig
    monkeypatch.setenv("RAC_QP_LL", ll)
    rng = np.random.default_rng(5)
    N, d, s = 1230, 12, 100
    X = rng.standard_normal((N, d))
    y = np.where(X[:, 0] + 0.3 * rng.standard_normal(N) > 0, 1.0, -1.0)
    want = {}
    ro.svm_train(X, y, C=1.0, block_size=s, beta=1.0, max_iters=6, seed=4, fixed_iterations=True,
                 on_sweep=lambda k, blocks, z, nu, primal, dual: want.__setitem__(k, (z.copy(), float(nu))))
    got = {}
    svm.train(X, y, 1.0, svm.KernelSpec("linear"),
              SolverConfig(block_size=s, beta_penalty=1.0, max_iters=6, seed=4, fixed_iterations=True),
              sweep_hook=lambda k, z, nu: got.__setitem__(k, (z, float(nu))))
    assert len(got) == len(want) == 6
    for k in want:
        assert rel(got[k][0], want[k][0]) <= ITER_TOL, (ll, k)
        assert abs(got[k][1] - want[k][1]) <= ITER_TOL * max(1.0, abs(want[k][1])), (ll, k)


def test_solve_invalid_problem(dev):
    from paper_1907_01995_b200 import engine
    from paper_1907_01995_b200.problems import QpProblem, SolverConfig
    prob = QpProblem(c=np.zeros(2), H=np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(ValueError, match="invalid problem"):
        engine.solve(prob, SolverConfig(block_size=1))


def test_solve_tiny_symmetric_qp_all_modes(dev):
    from paper_1907_01995_b200 import engine
    from paper_1907_01995_b200.problems import Mode, QpProblem, SolverConfig, Status
    for mode in (Mode.RAC, Mode.RP, Mode.CYCLIC):
        prob = QpProblem(c=np.zeros(2), H=np.eye(2), A=np.array([[1.0, 1.0]]), b=np.array([2.0]))
        res = engine.solve(prob, SolverConfig(mode=mode, block_size=1, beta_penalty=1.0, max_iters=500,
                                              tol_primal=1e-10, tol_dual=1e-10, seed=4))
        assert res.status == Status.CONVERGED
        np.testing.assert_allclose(res.x, [1.0, 1.0], atol=1e-8)
        np.testing.assert_allclose(res.y, [1.0], atol=1e-8)


def test_solve_determinism(dev):
    from paper_1907_01995_b200 import engine
    from paper_1907_01995_b200.problems import QpProblem, SolverConfig
    rng = np.random.default_rng(2)
    G = rng.standard_normal((40, 40))
    H = G @ G.T / 40 + 0.5 * np.eye(40)
    H = 0.5 * (H + H.T)
    A = rng.standard_normal((3, 40))
    prob = QpProblem(c=rng.standard_normal(40), H=H, A=A, b=A @ rng.uniform(-0.2, 0.2, 40),
                     lower=np.full(40, -0.3), upper=np.full(40, 0.3))
    cfg = SolverConfig(block_size=6, beta_penalty=0.7, max_iters=30, tol_primal=1e-16, tol_dual=1e-16,
                       seed=9, fixed_iterations=True)
    a, b = engine.solve(prob, cfg), engine.solve(prob, cfg)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y)
    assert np.array_equal(a.primal_residual_history, b.primal_residual_history)


# ---------------------------------------------------------------- svm.train
@pytest.mark.parametrize("strips", ["0", "1"])
@pytest.mark.parametrize("tag", ["lin", "gauss", "gauss_rp", "cfg4s"])
def test_train_matches_reference(dev, golden, tag, strips, monkeypatch):
    """strips=1: kernel strips formed on the fly per batch of blocks (the
    reference's own scheme) instead of the resident N x N matrix (rp keeps the matrix)."""
    from paper_1907_01995_b200 import svm
    from paper_1907_01995_b200.problems import Mode, SolverConfig
    monkeypatch.setenv("RAC_SVM_STRIPS", strips)
    monkeypatch.setattr(svm, "STRIP_BYTES", 1 << 14)     # several strip batches per sweep
    g = golden("svm_small")
    C, bs, beta, iters, tp, td, seed, fixed, sigma = g[f"{tag}_params"]
    cfg = SolverConfig(mode=Mode(str(g[f"{tag}_mode"])), block_size=int(bs), beta_penalty=float(beta),
                       max_iters=int(iters), tol_primal=float(tp), tol_dual=float(td), seed=int(seed),
                       fixed_iterations=bool(fixed))
    zs, nus = [], []
    model, diag = svm.train(g[f"{tag}_X"], g[f"{tag}_y"], float(C),
                            svm.KernelSpec(str(g[f"{tag}_kernel"]), float(sigma)), cfg,
                            return_diagnostics=True,
                            sweep_hook=lambda k, z, nu: (zs.append(z), nus.append(nu)))
    assert diag.iterations == int(g[f"{tag}_iterations"])
    assert diag.status.value == str(g[f"{tag}_status"])
    for k in range(min(diag.iterations, 50)):
        assert rel(zs[k], g[f"{tag}_z"][k]) <= ITER_TOL, (tag, k)
        assert abs(nus[k] - g[f"{tag}_nu"][k]) <= ITER_TOL * max(1.0, abs(g[f"{tag}_nu"][k])), (tag, k)
    np.testing.assert_allclose(diag.primal_residual_history, g[f"{tag}_primal"], rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(diag.dual_residual_history, g[f"{tag}_dual"], rtol=1e-6, atol=1e-12)
    # final dual objective 1/2 z'Qz - 1'z
    from oracle import rac_oracle as ro
    X, y = g[f"{tag}_X"], g[f"{tag}_y"]
    Q = (y[:, None] * ro.kernel_matrix(X, X, str(g[f"{tag}_kernel"]), float(sigma))) * y[None, :]
    want = ro.svm_dual_objective(Q, g[f"{tag}_z"][-1])
    got = ro.svm_dual_objective(Q, diag.duals)
    assert abs(got - want) <= OBJ_TOL * abs(want)
    assert abs(model.bias - float(g[f"{tag}_bias"])) <= 1e-7 * max(1.0, abs(float(g[f"{tag}_bias"])))


def test_train_validation(dev):
    from paper_1907_01995_b200 import svm
    X = np.zeros((3, 1))
    with pytest.raises(ValueError, match="labels"):
        svm.train(X, np.array([1.0, 2.0, -1.0]), 1.0, svm.KernelSpec("linear"))
    with pytest.raises(ValueError, match="C"):
        svm.train(X, np.array([1.0, 1.0, -1.0]), -1.0, svm.KernelSpec("linear"))


def test_build_q_matches_kernel_rows(dev):
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import svm
    rng = np.random.default_rng(3)
    X = rng.standard_normal((130, 7))
    y = np.where(rng.random(130) < 0.5, 1.0, -1.0)
    for kernel in (svm.KernelSpec("linear"), svm.KernelSpec("gaussian", 1.3)):
        Q = svm.build_q(X, y, kernel).cpu().numpy()
        want = (y[:, None] * ro.kernel_matrix(X, X, kernel.kind, kernel.sigma)) * y[None, :]
        assert np.max(np.abs(Q - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))
        assert np.array_equal(Q, Q.T)


def test_build_q_int8_tensor_cores(dev, monkeypatch):
    """RAC_Q_I8=2 forces Q = Y X X' Y onto the int8 digit-slice tensor-core Gram (the default
    once its tiles fill the SMs): ragged N and d, both kernels, against the oracle's kernel
    matrix; then a train on it matches the DMMA-built one to the parity bar."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import svm
    rng = np.random.default_rng(4)
    X = rng.standard_normal((333, 37))
    y = np.where(rng.random(333) < 0.5, 1.0, -1.0)
    for kernel in (svm.KernelSpec("linear"), svm.KernelSpec("gaussian", 1.1)):
        monkeypatch.setenv("RAC_Q_I8", "2")
        Q8 = svm.build_q(X, y, kernel).cpu().numpy()
        monkeypatch.setenv("RAC_Q_I8", "0")
        Q0 = svm.build_q(X, y, kernel).cpu().numpy()
        want = (y[:, None] * ro.kernel_matrix(X, X, kernel.kind, kernel.sigma)) * y[None, :]
        scale = max(1.0, np.max(np.abs(want)))
        assert np.max(np.abs(Q8 - want)) <= 1e-13 * scale
        assert np.max(np.abs(Q8 - Q0)) <= 1e-13 * scale
        assert np.array_equal(Q8, Q8.T)
