"""Pin the CPU oracle (oracle/rac_oracle.py) to the reference's own outputs.

The fixtures under tests/golden/ were produced by running the unmodified
reference racml (tests/golden/make_golden.py).  CPU-only.
"""

import hashlib

import numpy as np
import pytest

from oracle import rac_oracle as ro
from paper_1907_01995_b200 import configs


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


# ---------------------------------------------------------------- chunks
def test_sorted_chunks_match_reference(golden):
    g = golden("chunks")
    for key in [k for k in g if k.startswith("perm_")]:
        tag = key[len("perm_"):]
        chunks = ro.sorted_chunks(g[key], int(tag.split("_")[1]))
        assert np.array_equal(np.concatenate(chunks), g["flat_" + tag])
        assert np.array_equal([c.size for c in chunks], g["lens_" + tag])


def test_config_size_chunks_hash(golden):
    g = golden("chunks")
    for n, s in [(500, 50), (2000, 100), (5000, 200), (20000, 100), (100000, 500)]:
        rng = np.random.default_rng(0)
        for k in range(2):
            flat = np.concatenate(ro.sorted_chunks(rng.permutation(n), s))
            assert hashlib.sha256(flat.tobytes()).digest() == g[f"sha_{n}_{s}_{k}"].tobytes()


# ---------------------------------------------------------------- prox / block
def test_soft_threshold_literals():
    assert ro.neg_shrink(3.0, 1.0) == -2.0
    assert ro.neg_shrink(-3.0, 1.0) == 2.0
    assert ro.neg_shrink(0.5, 1.0) == 0.0
    assert np.signbit(ro.neg_shrink(0.5, 1.0)) == False  # noqa: E712  (-0 killed)


def test_prox_matches_reference(golden):
    g = golden("block_prox")
    assert np.array_equal(ro.neg_shrink(g["prox_a"], g["prox_b"]), g["prox_st"])
    assert np.array_equal(ro.z_prox(g["prox_beta"], g["prox_xi"], 0.7, 0.4, 0.3), g["prox_z"])


def test_box_block_min_matches_reference(golden):
    g = golden("block_prox")
    for i in range(int(g["blk_count"])):
        x = ro.box_block_min(g[f"blk{i}_M"], g[f"blk{i}_r"], g[f"blk{i}_lo"], g[f"blk{i}_hi"])
        np.testing.assert_array_equal(x, g[f"blk{i}_x"])


# ---------------------------------------------------------------- elastic net
def _en_params(g, tag):
    lam, alpha, gamma, bs, iters, seed, tol = g[f"{tag}_params"]
    return dict(lam=lam, alpha=alpha, gamma=None if np.isnan(gamma) else gamma,
                block_size=int(bs), iters=int(iters), seed=int(seed),
                tol=None if np.isnan(tol) else tol, mode=str(g[f"{tag}_mode"]))


def _check_en(g, tag, X, y):
    caps = {}
    res = ro.en_fit(X, y, **_en_params(g, tag),
                    on_sweep=lambda k, blocks, b, z, xi: caps.__setitem__(
                        k, (np.concatenate(blocks), b.copy(), z.copy(), xi.copy())))
    for k in g[f"{tag}_sweeps_kept"]:
        blocks, b, z, xi = caps[int(k)]
        if f"{tag}_blocks_{k}" in g:
            assert np.array_equal(blocks, g[f"{tag}_blocks_{k}"])
        assert rel(b, g[f"{tag}_beta_{k}"]) <= 1e-13
        assert rel(z, g[f"{tag}_z_{k}"]) <= 1e-13
        assert rel(xi, g[f"{tag}_xi_{k}"]) <= 1e-13
    gamma, iters, resid, obj_b, obj_z = g[f"{tag}_final"]
    assert res["iterations"] == int(iters)
    assert res["gamma"] == gamma
    assert rel(res["beta"], g[f"{tag}_final_beta"]) <= 1e-12
    assert abs(ro.en_objective(X, y, res["beta"], _en_params(g, tag)["lam"],
                               _en_params(g, tag)["alpha"]) - obj_b) <= 1e-12 * abs(obj_b)


@pytest.mark.parametrize("tag", ["lasso_rac", "ridge_rp", "enet_tol", "ls_lam0", "clamp_bs"])
def test_en_small_matches_reference(golden, tag):
    g = golden("en_small")
    _check_en(g, tag, g[f"{tag}_X"], g[f"{tag}_y"])


def test_en_config1_matches_reference(golden):
    g = golden("en_config1")
    c = configs.config1()
    _check_en(g, "cfg1", c.X, c.y)


def test_en_config2_small_matches_reference(golden):
    g = golden("en_config2_small")
    c = configs.config2(scale=0.1)
    _check_en(g, "cfg2s", c.X, c.y)


# ---------------------------------------------------------------- svm
@pytest.mark.parametrize("tag", ["lin", "gauss", "gauss_rp", "cfg4s"])
def test_svm_matches_reference(golden, tag):
    g = golden("svm_small")
    C, bs, beta, iters, tp, td, seed, fixed, sigma = g[f"{tag}_params"]
    zs, nus = [], []
    res = ro.svm_train(g[f"{tag}_X"], g[f"{tag}_y"], C, str(g[f"{tag}_kernel"]), sigma,
                       block_size=int(bs), beta=beta, max_iters=int(iters), tol_primal=tp,
                       tol_dual=td, seed=int(seed), mode=str(g[f"{tag}_mode"]),
                       fixed_iterations=bool(fixed),
                       on_sweep=lambda k, bl, z, nu, p, d: (zs.append(z.copy()), nus.append(nu)))
    assert res["iterations"] == int(g[f"{tag}_iterations"])
    assert res["status"] == str(g[f"{tag}_status"])
    for k in range(res["iterations"]):
        assert rel(zs[k], g[f"{tag}_z"][k]) <= 1e-12
        assert abs(nus[k] - g[f"{tag}_nu"][k]) <= 1e-12 * max(1.0, abs(g[f"{tag}_nu"][k]))
    np.testing.assert_allclose(res["primal_history"], g[f"{tag}_primal"], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(res["dual_history"], g[f"{tag}_dual"], rtol=1e-9, atol=1e-15)
    bias = ro.svm_bias(res["z"], g[f"{tag}_X"], g[f"{tag}_y"], C, str(g[f"{tag}_kernel"]), sigma)
    assert abs(bias - float(g[f"{tag}_bias"])) <= 1e-10 * max(1.0, abs(bias))


# ---------------------------------------------------------------- qp
@pytest.mark.parametrize("tag", ["box_rac", "box_rp", "free_cyclic", "medium_box", "h_only", "diverge"])
def test_qp_matches_reference(golden, tag):
    g = golden("qp_small")
    bs, beta, iters, tp, td, seed, fixed = g[f"{tag}_params"]
    xs, ys, orders = [], [], []
    res = ro.qp_solve(g[f"{tag}_c"], H=g.get(f"{tag}_H"), A=g.get(f"{tag}_A"), b=g.get(f"{tag}_b"),
                      lower=g[f"{tag}_lower"], upper=g[f"{tag}_upper"], mode=str(g[f"{tag}_mode"]),
                      block_size=int(bs), beta=beta, max_iters=int(iters), tol_primal=tp,
                      tol_dual=td, seed=int(seed), fixed_iterations=bool(fixed),
                      on_sweep=lambda k, bl, x, y: (xs.append(x.copy()), ys.append(y.copy()),
                                                    orders.append(np.concatenate(bl))))
    assert np.array_equal(orders[0], g[f"{tag}_order_1"])
    assert res["iterations"] == int(g[f"{tag}_iterations"])
    assert res["status"] == str(g[f"{tag}_status"])
    for k in range(min(res["iterations"], 50)):
        assert rel(xs[k], g[f"{tag}_x"][k]) <= 1e-12
        if ys[k].size:
            assert rel(ys[k], g[f"{tag}_y"][k]) <= 1e-12
    np.testing.assert_allclose(res["primal_history"][:50], g[f"{tag}_primal"][:50], rtol=1e-8, atol=1e-14)
    np.testing.assert_allclose(res["dual_history"][:50], g[f"{tag}_dual"][:50], rtol=1e-8, atol=1e-14)


def test_consensus_oracle_matches_reference(golden):
    """oracle.consensus_fit (restatement of elastic_net.py:252-316) vs the unmodified racml."""
    from oracle import rac_oracle as ro
    g = golden("consensus")
    for tag in ("direct", "woodbury", "mixed_tol", "ridge"):
        lam, alpha, gamma, bs, iters, seed, tol = g[f"{tag}_params"]
        r = ro.consensus_fit(g[f"{tag}_X"], g[f"{tag}_y"], lam, alpha, None if np.isnan(gamma) else gamma, int(bs),
                             int(iters), int(seed), None if np.isnan(tol) else tol)
        assert r["iterations"] == int(g[f"{tag}_final"][1])
        for k in ("beta", "z", "xi"):
            np.testing.assert_allclose(r[k], g[f"{tag}_{k}"], rtol=1e-12, atol=1e-14)


def test_full_size_fixtures_are_complete(golden):
    """The full-BASELINE-size fixtures (make_golden.py full2/3/4/5) hold what test_gpu_full
    needs: first-sweep blocks, iterates at sweeps 1, 2, 5, 10, 25, 50 (those reached), every
    sweep's norms, the final objective and iteration count."""
    for cfg, n, s in ((2, 2000, 100), (3, 5000, 200), (5, 100000, 500)):
        g = golden(f"en_config{cfg}_full")
        t = f"cfg{cfg}"
        assert np.array_equal(np.sort(g[f"{t}_blocks_1"]), np.arange(n))
        for k in g[f"{t}_sweeps_kept"]:
            assert g[f"{t}_beta_{int(k)}"].shape == (n,)
        assert g[f"{t}_norms"].shape[1] == 3 and g[f"{t}_final"].shape == (5,)
    assert int(golden("en_config2_full")["cfg2_final"][1]) == 43
    assert int(golden("en_config3_full")["cfg3_final"][1]) == 70
    assert int(golden("en_config5_full")["cfg5_final"][1]) == 50
    g = golden("svm_config4_full")
    assert int(g["cfg4_iterations"]) == 50 and g["cfg4_nu"].shape == (50,)
    assert np.array_equal(np.sort(g["cfg4_blocks_1"]), np.arange(20000))
    for k in g["cfg4_sweeps_kept"]:
        assert g[f"cfg4_z_{int(k)}"].shape == (20000,)


def _sparse_case(g, tag):
    import scipy.sparse as sps
    if tag == "ref":
        return sps.csc_matrix(g["ref_X"]), g["ref_y"]
    shp = tuple(int(v) for v in g["big_shape"])
    return sps.csc_matrix((g["big_data"], g["big_indices"], g["big_indptr"]), shape=shp), g["big_y"]


@pytest.mark.parametrize("tag", ["ref", "big"])
def test_sparse_oracle_matches_reference(golden, tag):
    """oracle.en_fit on CSC input (the reference densifies each block's columns) vs racml."""
    from oracle import rac_oracle as ro
    g = golden("en_sparse")
    X, y = _sparse_case(g, tag)
    lam, alpha, gamma, bs, iters, seed, tol = g[f"{tag}_params"]
    caps = {}
    ro.en_fit(X, y, lam, alpha, None if np.isnan(gamma) else gamma, int(bs), int(iters), seed=int(seed),
              on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
    for k in g[f"{tag}_sweeps_kept"]:
        b, z, xi = caps[int(k)]
        for got, key in ((b, "beta"), (z, "z"), (xi, "xi")):
            want = g[f"{tag}_{key}_{int(k)}"]
            assert np.linalg.norm(got - want) <= 1e-12 * max(np.linalg.norm(want), 1e-300)
