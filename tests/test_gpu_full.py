"""GPU parity at the FULL BASELINE sizes (north_star: "on one B200, every config matches the
CPU oracle"), against fixtures produced by the unmodified racml at the SURVEY §8(d)
seed-0 recipe (tests/golden/make_golden.py full2 / full3 / full4 / full5).

Inputs are regenerated from the seed (paper_1907_01995_b200.configs); the public entry
points run with their DEFAULT paths, i.e. exactly what the bench times:
  * config 2: covariance mode, G on the int8 tensor cores, lookahead chain, run to 1e-6;
  * config 3: covariance mode, int8 G over m = 50 000 samples (crosses the 65 472-sample
    int32 segment), s = 200 factor, run to 1e-6 (70 sweeps);
  * config 4: svm.train, Q = (YX)(YX)' on the int8 tensor cores (d = 500), 50 sweeps;
  * config 5: block mode, int8 block Grams at s = 500, the large-s blocked inverse,
    streaming chain, 50 sweeps.
Bars (north_star): block indices bit-exact; beta / z / xi (EN), z / nu (SVM) within 1e-9
relative L2 after every kept sweep (1, 2, 5, 10, 25, 50) and the norms of EVERY sweep
<= 50 within 1e-9 relative; final objective within 1e-8 relative; iteration counts +-1.
"""

import numpy as np
import pytest
import torch

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


def _first_sweep_blocks(n, s, seed):
    """Device chunk sort of the first RAC permutation (the reference's rng call order)."""
    from paper_1907_01995_b200 import _device, _native
    lib = _native.load()
    perm = np.random.default_rng(seed).permutation(n)
    p = -(-n // s)
    out = torch.empty(p * s, dtype=torch.int32, device="cuda")
    _native.check(lib.rac_chunk_sort(torch.from_numpy(perm).cuda().data_ptr(), n, s, 1, out.data_ptr(),
                                     _device.stream_handle()))
    got = out.cpu().numpy()
    return got[got >= 0]


@pytest.mark.parametrize("cfg", [2, 3, 5])
def test_fit_full_size_matches_reference(dev, golden, cfg):
    from paper_1907_01995_b200 import configs
    from paper_1907_01995_b200 import elastic_net as en
    g = golden(f"en_config{cfg}_full")
    tag = f"cfg{cfg}"
    lam, alpha, gamma, bs, iters, seed, tol = g[f"{tag}_params"]
    case = configs.GENERATORS[cfg]()
    assert (case.lam, case.alpha, case.block_size, case.seed) == (lam, alpha, int(bs), int(seed))
    spec = en.ElasticNetSpec(lam=float(lam), alpha=float(alpha), gamma=None if np.isnan(gamma) else float(gamma),
                             block_size=int(bs), iters=int(iters), seed=int(seed),
                             tol=None if np.isnan(tol) else float(tol))
    m, n = case.X.shape
    assert np.array_equal(_first_sweep_blocks(n, int(bs), int(seed)), g[f"{tag}_blocks_1"].astype(np.int64))
    kept = set(int(k) for k in g[f"{tag}_sweeps_kept"])
    norms, caps = [], {}

    def hook(k, b, z, xi):
        if k <= 50:
            norms.append((np.linalg.norm(b), np.linalg.norm(z), np.linalg.norm(xi)))
        if k in kept:
            caps[k] = (b.copy(), z.copy(), xi.copy())

    model = en.fit(case.X, case.y, spec, sweep_hook=hook)
    for k in sorted(kept):
        b, z, xi = caps[k]
        assert rel(b, g[f"{tag}_beta_{k}"]) <= ITER_TOL, (cfg, k, "beta", rel(b, g[f"{tag}_beta_{k}"]))
        assert rel(z, g[f"{tag}_z_{k}"]) <= ITER_TOL, (cfg, k, "z", rel(z, g[f"{tag}_z_{k}"]))
        assert rel(xi, g[f"{tag}_xi_{k}"]) <= ITER_TOL, (cfg, k, "xi", rel(xi, g[f"{tag}_xi_{k}"]))
    want = g[f"{tag}_norms"][:len(norms)]
    got = np.asarray(norms)
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)) <= ITER_TOL
    gm, it_ref, res_ref, obj_b, obj_z = g[f"{tag}_final"]
    assert abs(model.iterations - int(it_ref)) <= 1, (model.iterations, it_ref)
    assert model.gamma == gm
    ob = en.objective(case.X, case.y, model.beta, spec.lam, spec.alpha)
    oz = en.objective(case.X, case.y, model.z, spec.lam, spec.alpha)
    assert abs(ob - obj_b) <= OBJ_TOL * abs(obj_b), (ob, obj_b)
    assert abs(oz - obj_z) <= OBJ_TOL * abs(obj_z), (oz, obj_z)
    if model.iterations == int(it_ref):
        assert rel(model.beta, g[f"{tag}_final_beta"]) <= ITER_TOL


@pytest.mark.parametrize("strips", ["0", "1"])
def test_train_config4_full_size_matches_reference(dev, golden, strips, monkeypatch):
    """strips=1: no resident 20000 x 20000 Q; per sweep the blocks' H_bb and batches of strip
    rows."""
    from paper_1907_01995_b200 import configs, svm
    from paper_1907_01995_b200.problems import Mode, SolverConfig
    monkeypatch.setenv("RAC_SVM_STRIPS", strips)
    g = golden("svm_config4_full")
    C, bs, beta, max_iters, tp, td, seed, fixed, sigma = g["cfg4_params"]
    case = configs.config4()
    N = case.X.shape[0]
    assert np.array_equal(_first_sweep_blocks(N, int(bs), int(seed)), g["cfg4_blocks_1"].astype(np.int64))
    kept = set(int(k) for k in g["cfg4_sweeps_kept"])
    zs, nus, znorms = {}, [], []

    def hook(k, z, nu):
        nus.append(nu)
        znorms.append(np.linalg.norm(z))
        if k in kept:
            zs[k] = z.copy()

    cfg = SolverConfig(mode=Mode.RAC, block_size=int(bs), beta_penalty=float(beta), max_iters=int(max_iters),
                       tol_primal=float(tp), tol_dual=float(td), seed=int(seed), fixed_iterations=bool(fixed))
    _, diag = svm.train(case.X, case.labels, float(C), svm.KernelSpec("linear"), cfg, return_diagnostics=True,
                        sweep_hook=hook)
    assert diag.iterations == int(g["cfg4_iterations"])
    for k in sorted(kept):
        assert rel(zs[k], g[f"cfg4_z_{k}"]) <= ITER_TOL, (k, rel(zs[k], g[f"cfg4_z_{k}"]))
    nu_ref = g["cfg4_nu"]
    assert np.max(np.abs(np.asarray(nus) - nu_ref) / np.maximum(np.abs(nu_ref), 1e-300)) <= ITER_TOL
    zn = g["cfg4_znorms"]
    assert np.max(np.abs(np.asarray(znorms) - zn) / np.maximum(zn, 1e-300)) <= ITER_TOL
    # residual histories: the primal |t| is a difference of O(1) sums, compare absolutely at the
    # scale of the duals' sum
    scale = max(1.0, float(np.sum(np.abs(g[f"cfg4_z_{max(kept)}"]))))
    assert np.max(np.abs(diag.primal_residual_history - g["cfg4_primal"])) <= ITER_TOL * scale
    np.testing.assert_allclose(diag.dual_residual_history, g["cfg4_dual"], rtol=1e-7, atol=1e-9)
    z = diag.duals
    w = case.X.T @ (case.labels * z)
    obj = 0.5 * float(w @ w) - float(z.sum())
    want = float(g["cfg4_dual_objective"])
    assert abs(obj - want) <= OBJ_TOL * abs(want), (obj, want)
