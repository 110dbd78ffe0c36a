"""The covariance Gram on the tcgen05 int8 tensor cores (csrc/gram_i8.cu, exact digit
slices) against an extended-precision host product and the FP64 DMMA tiles."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1907_01995_b200 import _native
    return _native.load()


def _gram(lib, Xc, len_, n, div, method, G=None):
    from paper_1907_01995_b200 import _native
    if G is None:
        G = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    _native.check(lib.rac_gram_covariance(C.c_void_p(Xc.data_ptr()), Xc.shape[1], len_, n,
                                          C.c_void_p(G.data_ptr()), div, method))
    return G


def _device_cols(X):
    m, n = X.shape
    ld = (m + 31) // 32 * 32
    Xc = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    Xc[:, :m] = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    return Xc


def _worst(X, S):
    """Per-entry worst case of the digit truncation: 2^-52.8 (S = 8) / 2^-45.8 (S = 7) of
    max|x_j| max|x_k| per sample (gram_i8.cu), plus the FP64 combination's rounding."""
    mx = np.abs(X).max(axis=0)
    return 2.0 ** (-52.8 if S == 8 else -45.8) * X.shape[0] * np.outer(mx, mx)


# (m, n): ragged tiles (n not a multiple of 64 / 128), one sample stage, several int32
# segments (m > 65472 samples), a single feature; S = 7 slices is what Gaussian columns
# (max/rms <= 8) get, S = 8 is forced by RAC_I8_SLICES=8 (and chosen for wider columns)
@pytest.mark.parametrize("slices", [7, 8])
@pytest.mark.parametrize("m,n", [(64, 8), (77, 129), (1000, 300), (3000, 700), (70000, 150), (500, 1)])
def test_int8_slice_gram_accuracy(lib, monkeypatch, m, n, slices):
    if slices == 8:
        monkeypatch.setenv("RAC_I8_SLICES", "8")
    rng = np.random.default_rng(m + n)
    X = rng.standard_normal((m, n))
    if slices == 7 and m > 8:
        assert (np.abs(X).max(axis=0) <= 8 * np.sqrt((X * X).mean(axis=0))).all()
    Xl = X.astype(np.longdouble)
    R = Xl.T @ Xl
    nrm = np.sqrt(np.diag(R).astype(np.float64))
    Xc = _device_cols(X)
    G8 = _gram(lib, Xc, m, n, 1.0, 1).cpu().numpy()
    G0 = _gram(lib, Xc, m, n, 1.0, 0).cpu().numpy()
    scale = np.maximum(np.outer(nrm, nrm), 1e-300)
    err = np.abs((G8.astype(np.longdouble) - R)).astype(np.float64)
    e8 = (err / scale).max()
    e0 = (np.abs((G0.astype(np.longdouble) - R)).astype(np.float64) / scale).max()
    assert (err <= _worst(X, slices) + 2.3e-16 * np.abs(R).astype(np.float64)).all()
    if slices == 8:
        # 2 ulp of |x_j||x_k| (exact int32 sums; only the digit truncation below
        # 2^-52.8 of max|x_j|max|x_k| per sample and the final FP64 combination round)
        assert e8 <= 1e-15, e8
        assert e8 <= max(e0, 1e-15)
    else:
        # the FP64 DMMA tiles' level (2e-15 .. 2e-14 measured on these shapes)
        assert e8 <= 2e-14, e8
    assert np.array_equal(G8, G8.T)                 # each pair formed once, mirrored


@pytest.mark.parametrize("slices", [7, 8])
def test_int8_slice_gram_scaled_and_zero_columns(lib, monkeypatch, slices):
    """Per-feature power-of-two scales: columns 1e-30 .. 1e30 and an all-zero column."""
    if slices == 8:
        monkeypatch.setenv("RAC_I8_SLICES", "8")
    rng = np.random.default_rng(5)
    m, n = 2000, 260
    X = rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-30, 30, n)
    X[:, 0] = 0.0
    X[:, 7] = 0.0
    Xl = X.astype(np.longdouble)
    R = Xl.T @ Xl
    nrm = np.sqrt(np.diag(R).astype(np.float64))
    G8 = _gram(lib, _device_cols(X), m, n, 1.0, 1).cpu().numpy()
    scale = np.maximum(np.outer(nrm, nrm), 1e-300)
    assert (np.abs((G8.astype(np.longdouble) - R)).astype(np.float64) / scale).max() <= (4.5e-16 if slices == 8 else 2e-14)
    assert np.all(G8[0] == 0.0) and np.all(G8[:, 7] == 0.0)


def test_int8_wide_columns_get_eight_slices(lib, monkeypatch):
    """A column with max/rms between 8 and 256 keeps the digit slices (no DMMA fallback)
    but raises the 8-slice flag: every entry meets the S = 8 truncation bound, which the
    S = 7 slicing of this data would exceed."""
    rng = np.random.default_rng(21)
    m, n = 4000, 200
    X = rng.standard_normal((m, n))
    X[17, 3] = 40.0 * np.sqrt((X[:, 3] ** 2).mean())       # r_3 ~ 40
    Xl = X.astype(np.longdouble)
    R = Xl.T @ Xl
    G8 = _gram(lib, _device_cols(X), m, n, 1.0, 1).cpu().numpy()
    err = np.abs((G8.astype(np.longdouble) - R)).astype(np.float64)
    assert (err <= _worst(X, 8) + 2.3e-16 * np.abs(R).astype(np.float64)).all()
    nrm = np.sqrt(np.diag(R).astype(np.float64))
    rel = err / np.outer(nrm, nrm)
    rel[3, :] = rel[:, 3] = 0.0        # the wide column's own entries: 2^-52.8 r_3 r_k (checked above)
    assert rel.max() <= 1e-15          # the other entries at the S = 8 level (S = 7 gives ~5e-15)


def test_int8_slice_gram_divides_and_accumulates(lib):
    """div > 0 writes sum / div; div = 0 adds to G (the row-chunk streaming of fit)."""
    rng = np.random.default_rng(9)
    m, n = 4096, 333
    X = rng.standard_normal((m, n))
    Xc = _device_cols(X)
    full = _gram(lib, Xc, m, n, float(m), 1).cpu().numpy()
    G = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    half = m // 2
    _gram(lib, Xc[:, :half].contiguous(), half, n, 0.0, 1, G)
    _gram(lib, Xc[:, half:].contiguous(), m - half, n, 0.0, 1, G)
    acc = G.cpu().numpy() / m
    ref = (X.T @ X) / m
    assert np.abs(full - ref).max() <= 1e-14 * np.abs(ref).max()
    assert np.abs(acc - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("ingest", ["host", "device"])
def test_covariance_fit_with_int8_gram_vs_oracle(lib, monkeypatch, ingest):
    """RAC_G_I8=2 forces the tensor-core Gram at sizes below its SM-filling threshold:
    device-resident X (one launch) and host X streamed in row chunks (pieces of >= 4096
    samples summed into G, the last piece ragged), per-sweep iterates against the oracle."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import _device, elastic_net as en
    monkeypatch.setenv("RAC_G_I8", "2")
    rng = np.random.default_rng(23)
    for (m, n, s) in [(300, 200, 40), (9000, 600, 64)]:
        X = rng.standard_normal((m, n))
        y = X[:, :9] @ rng.standard_normal(9) + 0.05 * rng.standard_normal(m)
        kw = dict(lam=0.05, alpha=0.7, gamma=1.0, block_size=s, iters=8, seed=4)
        caps = {}
        ro.en_fit(X, y, mode="rac", **kw,
                  on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
        got = {}
        Xin = X if ingest == "host" else torch.from_numpy(X).cuda()
        if ingest == "host" and m == 9000:
            assert 8 * m * n > 2 * _device.ROW_CHUNK_BYTES      # the row-chunk path
        en.fit(Xin, y, en.ElasticNetSpec(**kw), gram_mode="covariance",
               sweep_hook=lambda k, b, z, xi: got.__setitem__(k, (b, z, xi)))
        for k in caps:
            for a_, b_ in zip(got[k], caps[k]):
                err = np.linalg.norm(a_ - b_) / max(np.linalg.norm(b_), 1e-300)
                assert err <= 1e-9, (m, n, s, k, err)


@pytest.mark.parametrize("ingest", ["host", "device"])
def test_block_mode_fit_with_int8_block_grams_vs_oracle(lib, monkeypatch, ingest):
    """RAC_BG_I8=2 forces the per-sweep int8 block Grams (gather-slicing of the partition's
    columns + one batched tensor-core launch) in block mode: short last block (padding),
    s above and below one 128-feature tile, rp mode; per-sweep iterates against the oracle."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    from paper_1907_01995_b200.problems import Mode
    monkeypatch.setenv("RAC_BG_I8", "2")
    rng = np.random.default_rng(31)
    for (m, n, s, mode) in [(400, 700, 150, "rac"), (9000, 520, 130, "rac"), (250, 300, 40, "rp")]:
        X = rng.standard_normal((m, n))
        y = X[:, :11] @ rng.standard_normal(11) + 0.05 * rng.standard_normal(m)
        kw = dict(lam=0.05, alpha=0.6, gamma=1.0, block_size=s, iters=6, seed=8)
        caps = {}
        ro.en_fit(X, y, mode=mode, **kw,
                  on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
        got = {}
        Xin = X if ingest == "host" else torch.from_numpy(X).cuda()
        en.fit(Xin, y, en.ElasticNetSpec(mode=Mode(mode), **kw), gram_mode="blocks",
               sweep_hook=lambda k, b, z, xi: got.__setitem__(k, (b, z, xi)))
        for k in caps:
            for a_, b_ in zip(got[k], caps[k]):
                err = np.linalg.norm(a_ - b_) / max(np.linalg.norm(b_), 1e-300)
                assert err <= 1e-9, (m, n, s, mode, k, err)


@pytest.mark.parametrize("gram,env", [("covariance", {}), ("blocks", {"RAC_BG_I8": "2"})])
def test_int8_grams_fall_back_on_heavy_outliers(lib, monkeypatch, gram, env):
    """A 1e12 outlier in a column leaves the digit slices ~1e-5 relative error in that column's
    Gram entries (the dropped products scale with max|x_j| max|x_k| per sample):
    the exponent pass flags the column (max/rms > 256) and the fit forms this data set's Grams
    on the FP64 DMMA tiles — per-sweep parity with the oracle holds."""
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import elastic_net as en
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(51)
    m, n, s = 3000, 1700, 170
    X = rng.standard_normal((m, n))
    X[17, 100] = 1e12
    X[400, 901] = -3e9
    y = X[:, :9] @ rng.standard_normal(9) + 0.05 * rng.standard_normal(m)
    kw = dict(lam=0.05, alpha=0.7, gamma=1.0, block_size=s, iters=4, seed=4)
    caps = {}
    ro.en_fit(X, y, mode="rac", **kw,
              on_sweep=lambda k, bl, b, z, xi: caps.__setitem__(k, (b.copy(), z.copy(), xi.copy())))
    got = {}
    en.fit(X, y, en.ElasticNetSpec(**kw), gram_mode=gram,
           sweep_hook=lambda k, b, z, xi: got.__setitem__(k, (b, z, xi)))
    for k in caps:
        for a_, b_ in zip(got[k], caps[k]):
            err = np.linalg.norm(a_ - b_) / max(np.linalg.norm(b_), 1e-300)
            assert err <= 1e-9, (gram, k, err)
    # the same context on well-behaved data goes back to the int8 tensor cores (flag reset)
    Xg = rng.standard_normal((m, n))
    a = en.fit(Xg, y, en.ElasticNetSpec(**kw), gram_mode=gram)
    r = ro.en_fit(Xg, y, mode="rac", **kw)
    assert np.linalg.norm(a.beta - r["beta"]) <= 1e-9 * np.linalg.norm(r["beta"])


def test_svm_q_falls_back_on_heavy_outliers(lib, monkeypatch):
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import svm
    from paper_1907_01995_b200.problems import Mode, SolverConfig
    monkeypatch.setenv("RAC_Q_I8", "2")
    rng = np.random.default_rng(52)
    N = 600
    lab = np.where(np.arange(N) < N // 2, 1.0, -1.0)
    X = rng.standard_normal((N, 40)) + lab[:, None] * 0.4
    X[7, 3] = 1e9
    cfg = SolverConfig(mode=Mode.RAC, block_size=50, beta_penalty=1.0, max_iters=3, seed=0)
    _, diag = svm.train(X, lab, 1.0, svm.KernelSpec("linear"), cfg, return_diagnostics=True)
    r = ro.svm_train(X, lab, 1.0, "linear", block_size=50, beta=1.0, max_iters=3, seed=0)
    assert np.linalg.norm(diag.duals - r["z"]) <= 1e-9 * max(np.linalg.norm(r["z"]), 1e-300)
