"""Accuracy and speed of the covariance Gram: int8 digit slices on tcgen05 (method 1)
against the FP64 DMMA tiles (method 0) and an extended-precision host reference."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_01995_b200 import _native

lib = _native.load()


def gram(Xc, len_, n, div, method, G=None):
    if G is None:
        G = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    rc = lib.rac_gram_covariance(C.c_void_p(Xc.data_ptr()), Xc.shape[1], len_, n, C.c_void_p(G.data_ptr()), div, method)
    _native.check(rc)
    return G


def ref(X):
    Xl = X.astype(np.longdouble)
    return (Xl.T @ Xl)


def check(m, n, seed=0, scale_cols=False, div=0.0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((m, n))
    if scale_cols:
        X *= 10.0 ** rng.uniform(-30, 30, n)
        X[:, 0] = 0.0
    ld = (m + 31) // 32 * 32
    Xc = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    Xc[:, :m] = torch.from_numpy(X.T.copy()).cuda()
    R = ref(X)
    nrm = np.sqrt(np.diag(R).astype(np.float64))
    out = {}
    for meth in (0, 1):
        G = gram(Xc, m, n, 1.0, meth).cpu().numpy()
        err = np.abs((G.astype(np.longdouble) - R).astype(np.float64)) / np.maximum(np.outer(nrm, nrm), 1e-300)
        out[meth] = (err.max(), np.abs(G - G.T).max())
    print(f"m={m} n={n} cols_scaled={scale_cols}: dmma err/(|xj||xk|) {out[0][0]:.2e} asym {out[0][1]:.1e} | "
          f"i8 {out[1][0]:.2e} asym {out[1][1]:.1e}", flush=True)


for (m, n) in [(64, 8), (77, 129), (1000, 300), (3000, 700), (70000, 150)]:
    check(m, n)
check(2000, 260, scale_cols=True)

for (m, n) in [(10000, 2000), (50000, 5000), (2000, 500)]:
    Xc = torch.randn((n, m), dtype=torch.float64, device="cuda")
    G = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    for meth in (0, 1):
        for _ in range(2):
            gram(Xc, m, n, float(m), meth, G)
        torch.cuda.synchronize()
        t = time.perf_counter()
        reps = 5
        for _ in range(reps):
            gram(Xc, m, n, float(m), meth, G)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / reps
        print(f"timing m={m} n={n} method={meth}: {dt*1e3:.3f} ms (incl. ws alloc + sync)", flush=True)
