"""GPU parity: elastic-net engine (fit) vs the reference's golden fixtures and the oracle.

Bars (BASELINE.json north_star): block indices bit-exact; iterates <= 1e-9
relative L2 after every sweep for the first 50 sweeps; final objective
<= 1e-8 relative.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-9      # relative L2, per sweep (north_star)
OBJ_TOL = 1e-8       # relative, final objective (north_star)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


@pytest.fixture(scope="module")
def lib():
    from paper_1907_01995_b200 import _device, _native
    _device.require_cuda(0)
    return _native.load()


def test_library_loaded_from_tree(lib):
    from paper_1907_01995_b200 import _native
    assert _native.MISSING == []
    with open("/proc/self/maps") as f:
        assert "librac_b200.so" in f.read()


def test_chunk_sort_bit_exact(lib, golden):
    from paper_1907_01995_b200 import _device, _native
    g = golden("chunks")
    for key in [k for k in g if k.startswith("perm_")]:
        tag = key[len("perm_"):]
        n, s = int(tag.split("_")[0]), int(tag.split("_")[1])
        perm = torch.from_numpy(g[key]).cuda()
        p = -(-n // s)
        out = torch.empty(p * s, dtype=torch.int32, device="cuda")
        _native.check(lib.rac_chunk_sort(perm.data_ptr(), n, s, 1, out.data_ptr(),
                                         _device.stream_handle()))
        got = out.cpu().numpy()
        got = got[got >= 0].astype(np.int64)
        assert np.array_equal(got, g["flat_" + tag])


def test_chunk_sort_config_sizes_bit_exact(lib):
    """Device chunk-sort vs the oracle's sorted chunks at every BASELINE (n, s), 3 sweeps each."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import _device, _native
    for n, s in [(500, 50), (2000, 100), (5000, 200), (20000, 100), (100000, 500), (1001, 7)]:
        rng = np.random.default_rng(0)
        perms = np.stack([rng.permutation(n) for _ in range(3)])
        p = -(-n // s)
        out = torch.empty(3 * p * s, dtype=torch.int32, device="cuda")
        _native.check(lib.rac_chunk_sort(torch.from_numpy(perms).cuda().data_ptr(), n, s, 3,
                                         out.data_ptr(), _device.stream_handle()))
        got = out.cpu().numpy().reshape(3, p * s)
        for k in range(3):
            want = np.concatenate(ro.sorted_chunks(perms[k], s))
            row = got[k]
            assert np.array_equal(row[row >= 0], want)


def test_z_prox_bit_exact(lib, golden):
    from paper_1907_01995_b200 import elastic_net as en
    g = golden("block_prox")
    z = en.z_update(torch.from_numpy(g["prox_beta"]).cuda(), torch.from_numpy(g["prox_xi"]).cuda(),
                    0.7, 0.4, 0.3)
    assert np.array_equal(z.cpu().numpy(), g["prox_z"])


def _spec_from(g, tag):
    from paper_1907_01995_b200.elastic_net import ElasticNetSpec
    from paper_1907_01995_b200.problems import Mode
    lam, alpha, gamma, bs, iters, seed, tol = g[f"{tag}_params"]
    return ElasticNetSpec(lam=float(lam), alpha=float(alpha),
                          gamma=None if np.isnan(gamma) else float(gamma),
                          block_size=int(bs), iters=int(iters), mode=Mode(str(g[f"{tag}_mode"])),
                          seed=int(seed), tol=None if np.isnan(tol) else float(tol))


def _check_fit(g, tag, X, y, check_all_sweeps=True, gram_mode="auto"):
    from paper_1907_01995_b200 import elastic_net as en
    spec = _spec_from(g, tag)
    caps = {}
    hook = (lambda k, b, z, xi: caps.__setitem__(k, (b, z, xi))) if check_all_sweeps else None
    model = en.fit(X, y, spec, sweep_hook=hook, gram_mode=gram_mode)
    gamma, iters, resid, obj_b, obj_z = g[f"{tag}_final"]
    if check_all_sweeps:
        for k in g[f"{tag}_sweeps_kept"]:
            k = int(k)
            if k > 50:
                continue
            b, z, xi = caps[k]
            assert rel(b, g[f"{tag}_beta_{k}"]) <= ITER_TOL, (tag, k)
            assert rel(z, g[f"{tag}_z_{k}"]) <= ITER_TOL, (tag, k)
            assert rel(xi, g[f"{tag}_xi_{k}"]) <= ITER_TOL, (tag, k)
    assert abs(model.iterations - int(iters)) <= 1, (model.iterations, iters)
    assert model.gamma == gamma
    got_obj = en.objective(X, y, model.beta, spec.lam, spec.alpha)
    assert abs(got_obj - obj_b) <= OBJ_TOL * abs(obj_b), (got_obj, obj_b)
    return model


@pytest.mark.parametrize("gram", ["blocks", "covariance"])
@pytest.mark.parametrize("tag", ["lasso_rac", "ridge_rp", "enet_tol", "ls_lam0", "clamp_bs"])
def test_fit_small_matches_reference(lib, golden, tag, gram):
    g = golden("en_small")
    _check_fit(g, tag, g[f"{tag}_X"], g[f"{tag}_y"], gram_mode=gram)


@pytest.mark.parametrize("gram", ["blocks", "covariance"])
def test_fit_config1_matches_reference(lib, golden, gram):
    from paper_1907_01995_b200 import configs
    g = golden("en_config1")
    c = configs.config1()
    _check_fit(g, "cfg1", c.X, c.y, gram_mode=gram)
    # norms of every one of the first 50 sweeps
    from paper_1907_01995_b200 import elastic_net as en
    caps = []
    en.fit(c.X, c.y, _spec_from(g, "cfg1"), sweep_hook=lambda k, b, z, xi: caps.append(
        (np.linalg.norm(b), np.linalg.norm(z), np.linalg.norm(xi))) if k <= 50 else None)
    got = np.asarray(caps)
    want = g["cfg1_norms"][:50]
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)) <= ITER_TOL


def test_fit_config2_small_matches_reference(lib, golden):
    from paper_1907_01995_b200 import configs
    g = golden("en_config2_small")
    c = configs.config2(scale=0.1)
    _check_fit(g, "cfg2s", c.X, c.y, gram_mode="blocks")
    _check_fit(g, "cfg2s", c.X, c.y, gram_mode="covariance")


def test_fit_vs_oracle_random_shapes(lib):
    """Ragged shapes (n % s != 0, m not a multiple of 32, s > 256) against the oracle."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    from paper_1907_01995_b200.problems import Mode
    rng = np.random.default_rng(7)
    # (3000, 600, 300): the one-tile streaming chain's last CTA owns fewer rows than the
    # others (regression: its row reductions overflowed the buffer sized for the full rows)
    for (m, n, s, mode, alpha) in [(33, 70, 9, "rac", 1.0), (257, 600, 300, "rac", 0.5), (3000, 600, 300, "rac", 0.8),
                                   (100, 513, 64, "rp", 0.2), (1, 5, 2, "rac", 1.0),
                                   (70, 20, 20, "rp", 0.0)]:
        X = rng.standard_normal((m, n))
        y = rng.standard_normal(m)
        kw = dict(lam=0.05, alpha=alpha, gamma=0.7, block_size=s, iters=12, seed=3)
        caps = {}
        ro.en_fit(X, y, mode=mode, **kw,
                  on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
        got = {}
        en.fit(X, y, en.ElasticNetSpec(mode=Mode(mode), **kw),
               sweep_hook=lambda k, b, z, xi: got.__setitem__(k, (b, z, xi)))
        for k in caps:
            for a_, b_ in zip(got[k], caps[k]):
                assert rel(a_, b_) <= ITER_TOL, (m, n, s, mode, k)


def test_fit_determinism(lib):
    from paper_1907_01995_b200 import elastic_net as en
    rng = np.random.default_rng(14)
    X = rng.standard_normal((250, 120))
    y = rng.standard_normal(250)
    spec = en.ElasticNetSpec(lam=0.1, alpha=0.8, block_size=25, iters=20, seed=21)
    a, b = en.fit(X, y, spec), en.fit(X, y, spec)
    assert np.array_equal(a.beta, b.beta) and np.array_equal(a.z, b.z) and np.array_equal(a.xi, b.xi)


def test_fit_validation_errors(lib):
    from paper_1907_01995_b200 import elastic_net as en
    from paper_1907_01995_b200.problems import Mode
    with pytest.raises(ValueError):
        en.fit(np.eye(2), np.zeros(2), en.ElasticNetSpec(lam=-1.0, alpha=0.5))
    with pytest.raises(ValueError):
        en.fit(np.eye(2), np.zeros(2), en.ElasticNetSpec(lam=1.0, alpha=2.0))
    with pytest.raises(ValueError):
        en.fit(np.eye(2), np.zeros(2), en.ElasticNetSpec(lam=1.0, alpha=0.5, mode=Mode.CYCLIC))
    with pytest.raises(ValueError):
        en.fit(np.eye(2), np.zeros(3), en.ElasticNetSpec(lam=1.0, alpha=0.5))


def test_identity_design_recovers_targets(lib):
    from paper_1907_01995_b200 import elastic_net as en
    n = 8
    y = np.arange(1.0, n + 1)
    model = en.fit(np.eye(n), y, en.ElasticNetSpec(lam=0.0, alpha=1.0, gamma=1.0, block_size=3,
                                                   iters=300, seed=1))
    np.testing.assert_allclose(model.beta, y, atol=1e-10)


@pytest.mark.parametrize("env,gram", [({}, "blocks"), ({"RAC_EN_PIPE": "0"}, "blocks"),
                                      ({"RAC_EN_CS": "4"}, "blocks"), ({"RAC_EN_CS": "8"}, "blocks"),
                                      ({"RAC_EN_VARIANT": "0"}, "blocks"), ({}, "covariance"),
                                      ({"RAC_EN_PIPE": "0"}, "covariance"),
                                      ({"RAC_COV_FULL": "0"}, "covariance")])
def test_chain_variants_match_oracle(lib, monkeypatch, env, gram):
    """Every chain variant (sweep pipeline on/off, cluster sizes 2/4/8, streaming chain,
    covariance chain) on a shape with several 32-row chunks per CTA, batched sweeps."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(31)
    m, n, s = 6000, 300, 60
    X = rng.standard_normal((m, n))
    y = X[:, :10] @ rng.standard_normal(10) + 0.1 * rng.standard_normal(m)
    kw = dict(lam=0.02, alpha=0.7, gamma=1.0, block_size=s, iters=25, seed=5)
    ref = ro.en_fit(X, y, mode="rac", **kw)
    got = en.fit(X, y, en.ElasticNetSpec(**kw), gram_mode=gram)
    assert rel(got.beta, ref["beta"]) <= ITER_TOL
    assert rel(got.z, ref["z"]) <= ITER_TOL
    assert rel(got.xi, ref["xi"]) <= ITER_TOL


def test_pipeline_bitwise_equals_serial(lib, monkeypatch):
    """Block mode: the cross-stream sweep pipeline runs the same kernels on the same data,
    bit-identical.  Covariance mode: the pipelined run chains a batch of sweeps in one
    launch (cross-sweep lookahead), so it equals the one-sweep-per-launch run to rounding."""
    from paper_1907_01995_b200 import elastic_net as en
    rng = np.random.default_rng(32)
    X = rng.standard_normal((3000, 400))
    y = rng.standard_normal(3000)
    spec = en.ElasticNetSpec(lam=0.05, alpha=0.9, block_size=40, iters=30, seed=9)
    for gram in ("blocks", "covariance"):
        monkeypatch.delenv("RAC_EN_PIPE", raising=False)
        a = en.fit(X, y, spec, gram_mode=gram)
        monkeypatch.setenv("RAC_EN_PIPE", "0")
        b = en.fit(X, y, spec, gram_mode=gram)
        if gram == "blocks":
            assert np.array_equal(a.beta, b.beta) and np.array_equal(a.z, b.z) and np.array_equal(a.xi, b.xi)
            assert np.array_equal(a.residual_history, b.residual_history)
        else:
            assert rel(a.beta, b.beta) <= ITER_TOL and rel(a.z, b.z) <= ITER_TOL and rel(a.xi, b.xi) <= ITER_TOL
            assert rel(a.residual_history, b.residual_history) <= 1e-6
    monkeypatch.delenv("RAC_EN_PIPE", raising=False)
    a = en.fit(X, y, spec, gram_mode="blocks")
    b = en.fit(X, y, spec, gram_mode="covariance")
    assert rel(a.beta, b.beta) <= ITER_TOL


@pytest.mark.parametrize("full", ["1", "0"])
def test_covariance_mode_vs_oracle_shapes(lib, monkeypatch, full):
    """Covariance chain on ragged shapes: n % s != 0, odd s (cp.async inverse path),
    n smaller than the cluster, rp mode, m < n, per-sweep parity for the first sweeps."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    from paper_1907_01995_b200.problems import Mode
    monkeypatch.setenv("RAC_COV_FULL", full)
    rng = np.random.default_rng(17)
    for (m, n, s, mode, alpha) in [(33, 70, 9, "rac", 1.0), (400, 600, 37, "rac", 0.5),
                                   (100, 513, 64, "rp", 0.2), (5, 7, 2, "rac", 1.0),
                                   (70, 20, 20, "rp", 0.0), (300, 1000, 256, "rac", 0.8)]:
        X = rng.standard_normal((m, n))
        y = rng.standard_normal(m)
        kw = dict(lam=0.05, alpha=alpha, gamma=0.7, block_size=s, iters=12, seed=3)
        caps = {}
        ro.en_fit(X, y, mode=mode, **kw,
                  on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
        got = {}
        en.fit(X, y, en.ElasticNetSpec(mode=Mode(mode), **kw), gram_mode="covariance",
               sweep_hook=lambda k, b, z, xi: got.__setitem__(k, (b, z, xi)))
        for k in caps:
            for a_, b_ in zip(got[k], caps[k]):
                assert rel(a_, b_) <= ITER_TOL, (m, n, s, mode, k)



@pytest.mark.parametrize("gram", ["blocks", "covariance"])
def test_streamed_ingest_matches_resident_input(lib, gram):
    """Host X above the streaming threshold goes through rac_en_set_data_rows (row chunks
    overlapping transfer, transpose and G += X_k'X_k); the same X as a device tensor goes
    through rac_en_set_data.  Block mode: bitwise equal; covariance mode: G is summed by
    chunks, so equal to rounding; both within the parity bar of the oracle."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import _device, elastic_net as en
    rng = np.random.default_rng(41)
    m, n = 5000, 1000
    assert 8 * m * n > 2 * _device.ROW_CHUNK_BYTES
    X = rng.standard_normal((m, n))
    y = X[:, :20] @ rng.standard_normal(20) + 0.1 * rng.standard_normal(m)
    spec = en.ElasticNetSpec(lam=0.05, alpha=0.8, gamma=1.0, block_size=100, iters=15, seed=2)
    a = en.fit(X, y, spec, gram_mode=gram)
    b = en.fit(torch.from_numpy(X).cuda(), y, spec, gram_mode=gram)
    if gram == "blocks":
        assert np.array_equal(a.beta, b.beta) and np.array_equal(a.z, b.z)
    else:
        assert rel(a.beta, b.beta) <= 1e-12
    ref = ro.en_fit(X, y, mode="rac", lam=0.05, alpha=0.8, gamma=1.0, block_size=100, iters=15, seed=2)
    assert rel(a.beta, ref["beta"]) <= ITER_TOL


@pytest.mark.parametrize("depth", ["1", "2", "3"])
def test_lookahead_chain_vs_oracle_shapes(lib, monkeypatch, depth):
    """Lookahead covariance chain (en_cla.cuh; even n and s): padded last block (n % s != 0),
    fewer 32-column segments than a worker cluster, rp mode (tiles follow the visit order),
    s > 128 (16-rank leader cluster), p >= 8 (tile-slot ring wraps), every lookahead depth;
    per-sweep iterates against the oracle."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    from paper_1907_01995_b200.problems import Mode
    monkeypatch.setenv("RAC_CLA_D", depth)
    rng = np.random.default_rng(23)
    for (m, n, s, mode, alpha) in [(500, 610, 40, "rac", 0.6), (200, 96, 12, "rac", 1.0),
                                   (300, 420, 30, "rp", 0.3), (400, 600, 150, "rac", 0.9),
                                   (120, 64, 64, "rac", 0.5), (260, 2000, 100, "rac", 1.0)]:
        X = rng.standard_normal((m, n))
        y = X[:, :5] @ rng.standard_normal(5) + 0.1 * rng.standard_normal(m)
        kw = dict(lam=0.05, alpha=alpha, gamma=0.8, block_size=s, iters=9, seed=4)
        caps = {}
        ro.en_fit(X, y, mode=mode, **kw,
                  on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
        got = {}
        en.fit(X, y, en.ElasticNetSpec(mode=Mode(mode), **kw), gram_mode="covariance",
               sweep_hook=lambda k, b, z, xi: got.__setitem__(k, (b, z, xi)))
        for k in caps:
            for a_, b_ in zip(got[k], caps[k]):
                assert rel(a_, b_) <= ITER_TOL, (m, n, s, mode, k)


def test_lookahead_chain_determinism_and_previous_form(lib, monkeypatch):
    """Batched sweeps through the lookahead chain are bit-identical run to run and agree
    with the previous single-cluster covariance chain (RAC_COV_LA=0) to the parity bar."""
    from paper_1907_01995_b200 import elastic_net as en
    rng = np.random.default_rng(29)
    X = rng.standard_normal((2000, 800))
    y = X[:, :8] @ rng.standard_normal(8) + 0.1 * rng.standard_normal(2000)
    spec = en.ElasticNetSpec(lam=0.05, alpha=0.8, block_size=50, iters=40, seed=6)
    a = en.fit(X, y, spec, gram_mode="covariance")
    b = en.fit(X, y, spec, gram_mode="covariance")
    assert np.array_equal(a.beta, b.beta) and np.array_equal(a.z, b.z) and np.array_equal(a.xi, b.xi)
    assert np.array_equal(a.residual_history, b.residual_history)
    monkeypatch.setenv("RAC_COV_LA", "0")
    c = en.fit(X, y, spec, gram_mode="covariance")
    assert rel(a.beta, c.beta) <= ITER_TOL and rel(a.z, c.z) <= ITER_TOL


@pytest.mark.parametrize("batch", [3, 5, 16])
def test_lookahead_batches_stop_at_the_converged_sweep(lib, batch):
    """Multi-sweep chain launches with a tolerance run the sweeps after the converging one
    speculatively and restore its snapshot: iteration count, residual history and the
    returned iterates are those of the oracle stopping at that sweep, for every offset of
    the converging sweep within a launch (fit batch sizes 3, 5, 16 host-side)."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    rng = np.random.default_rng(37)
    m, n, s = 3000, 600, 30
    X = rng.standard_normal((m, n))
    y = X[:, :6] @ rng.standard_normal(6) + 0.01 * rng.standard_normal(m)
    kw = dict(lam=0.02, alpha=1.0, gamma=1.0, block_size=s, iters=400, seed=8, tol=1e-7)
    ref = ro.en_fit(X, y, mode="rac", **kw)
    got = en.fit(X, y, en.ElasticNetSpec(**kw), gram_mode="covariance", batch=batch)
    assert abs(got.iterations - ref["iterations"]) <= 1
    assert len(got.residual_history) == got.iterations and got.residual_history[-1] == got.residual
    assert got.residual <= kw["tol"] and np.all(got.residual_history[:-1] > kw["tol"])
    if got.iterations == ref["iterations"]:
        assert abs(got.residual - ref["residual"]) <= 1e-6 * abs(ref["residual"])
        assert rel(got.beta, ref["beta"]) <= ITER_TOL and rel(got.z, ref["z"]) <= ITER_TOL
        assert rel(got.xi, ref["xi"]) <= ITER_TOL


@pytest.mark.parametrize("one_tile", ["1", "0"])
def test_streaming_chain_one_tile_vs_oracle(lib, monkeypatch, one_tile):
    """Block mode with s > 256 runs the streaming chain: one-tile resident row phase
    (RAC_EN_1T=1, CTAs own contiguous rows; the last CTA's range is short) and the
    chunked schedule (RAC_EN_1T=0), per-sweep iterates against the oracle."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    monkeypatch.setenv("RAC_EN_1T", one_tile)
    rng = np.random.default_rng(43)
    for (m, n, s, alpha) in [(500, 1200, 300, 1.0), (1000, 900, 300, 0.5), (150, 640, 320, 0.9)]:
        X = rng.standard_normal((m, n))
        y = X[:, :7] @ rng.standard_normal(7) + 0.05 * rng.standard_normal(m)
        kw = dict(lam=0.05, alpha=alpha, gamma=1.0, block_size=s, iters=6, seed=2)
        caps = {}
        ro.en_fit(X, y, mode="rac", **kw,
                  on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
        got = {}
        en.fit(X, y, en.ElasticNetSpec(**kw), gram_mode="blocks",
               sweep_hook=lambda k, b, z, xi: got.__setitem__(k, (b, z, xi)))
        for k in caps:
            for a_, b_ in zip(got[k], caps[k]):
                assert rel(a_, b_) <= ITER_TOL, (m, n, s, k)


@pytest.mark.parametrize("handoffs", ["0", "1", "9"])
def test_streaming_chain_tagged_handoffs_vs_oracle(lib, monkeypatch, handoffs):
    """The one-tile streaming chain with three grid barriers per block (RAC_EN_LL=0), with the row
    phase's partials handed to S1 as tagged words the reader spins on (1), and with the fused S
    phase on top (9, the default: one grid barrier per block): each gives the oracle's per-sweep
    iterates, also when the pooled context is used again (the tags of a new launch must not match
    the words a previous fit left behind) and with a short last block."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    monkeypatch.setenv("RAC_EN_LL", handoffs)
    rng = np.random.default_rng(47)
    for (m, n, s, alpha) in [(700, 1000, 300, 0.9), (150, 650, 320, 1.0)]:
        for rep in range(2):
            X = rng.standard_normal((m, n))
            y = X[:, :5] @ rng.standard_normal(5) + 0.05 * rng.standard_normal(m)
            kw = dict(lam=0.05, alpha=alpha, gamma=1.0, block_size=s, iters=5, seed=3 + rep)
            caps = {}
            ro.en_fit(X, y, mode="rac", **kw,
                      on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
            got = {}
            en.fit(X, y, en.ElasticNetSpec(**kw), gram_mode="blocks",
                   sweep_hook=lambda k, b, z, xi: got.__setitem__(k, (b, z, xi)))
            for k in caps:
                for a_, b_ in zip(got[k], caps[k]):
                    assert rel(a_, b_) <= ITER_TOL, (handoffs, m, n, s, rep, k)
            # without the per-sweep hook: several sweeps per run call, same final iterate
            fin = en.fit(X, y, en.ElasticNetSpec(**kw), gram_mode="blocks")
            assert rel(fin.beta, caps[max(caps)][0]) <= ITER_TOL


@pytest.mark.parametrize("gram", ["covariance", "blocks"])
def test_fit_enqueue_ahead_stops_where_the_synchronous_loop_does(lib, gram):
    """fit() with a tolerance enqueues batch k+1 before polling batch k (rac_en_poll); the
    speculative batch after convergence must be a no-op: same iterations, residual and
    iterates as the per-sweep synchronous loop (sweep_hook path) and as the oracle."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    rng = np.random.default_rng(12)
    m, n, s = 600, 240, 24
    X = rng.standard_normal((m, n))
    y = X[:, :6] @ rng.standard_normal(6) + 0.01 * rng.standard_normal(m)
    spec = en.ElasticNetSpec(lam=0.05, alpha=0.9, gamma=1.0, block_size=s, iters=500, seed=5, tol=1e-6)
    fast = en.fit(X, y, spec, gram_mode=gram, batch=16)
    slow = en.fit(X, y, spec, gram_mode=gram, sweep_hook=lambda *a: None)
    ref = ro.en_fit(X, y, mode="rac", lam=0.05, alpha=0.9, gamma=1.0, block_size=s, iters=500, seed=5, tol=1e-6)
    assert fast.iterations == slow.iterations == ref["iterations"] < 500
    # one sweep per launch (hook) vs batched launches: equal to rounding
    assert rel(fast.beta, slow.beta) <= 1e-12 and rel(fast.xi, slow.xi) <= 1e-12
    assert abs(fast.residual - slow.residual) <= 1e-9 * max(slow.residual, 1e-300)
    assert rel(fast.beta, ref["beta"]) <= ITER_TOL


@pytest.mark.parametrize("gram", ["blocks", "covariance"])
@pytest.mark.parametrize("tag", ["ref", "big"])
def test_fit_sparse_csc_matches_reference(lib, golden, tag, gram):
    """Sparse X: the CSC arrays go to the device and are expanded there;
    per-sweep iterates against racml's sparse column-block fit (golden en_sparse)."""
    import scipy.sparse as sps
    from paper_1907_01995_b200 import elastic_net as en
    g = golden("en_sparse")
    if tag == "ref":
        X, y = sps.csc_matrix(g["ref_X"]), g["ref_y"]
    else:
        X = sps.csc_matrix((g["big_data"], g["big_indices"], g["big_indptr"]),
                           shape=tuple(int(v) for v in g["big_shape"]))
        y = g["big_y"]
    _check_fit(g, tag, X, y, gram_mode=gram)
    # CSR / COO inputs go through the same canonical CSC
    spec = _spec_from(g, tag)
    a = en.fit(X.tocsr(), y, spec, gram_mode=gram)
    b = en.fit(X, y, spec, gram_mode=gram)
    assert np.array_equal(a.beta, b.beta)
