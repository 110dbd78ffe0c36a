"""C-SVC dual QP by RAC block sweeps on one B200 — drop-in for racml.svm.train.

    min 1/2 z'Qz - 1'z   s.t.  y'z = 0,  0 <= z <= C,   Q_ij = y_i y_j K(x_i, x_j)

The label-weighted kernel matrix is built once on the device with FP64
tensor-core tiles (`rac_svm_build_q`), then the dense box-QP engine runs the
sweep with H = Q, A = y', b = 0, c = -1 and the reference's 1e-9 relative
ridge (svm.py:241-246).  Same signature, validation, defaults, SvmModel and
TrainDiagnostics as svm.py:37-284.  `cache_capacity` is accepted for
signature compatibility; the device keeps all of Q resident instead of an
LRU of kernel rows.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.sparse as sp
import torch

from . import _device, _native
from .engine import QpSolver, drive
from .problems import Matrix, Mode, SolverConfig, Status

SUPPORT_THRESHOLD = 1e-8   # svm.py:25
MARGIN_DELTA = 1e-6        # svm.py:26
RIDGE_REL = 1e-9           # svm.py:245


class DegenerateModelError(RuntimeError):
    """No support vectors (svm.py:29-30)."""


@dataclass(frozen=True)
class KernelSpec:
    """Kernel choice (svm.py:37-48)."""

    kind: str = "gaussian"
    sigma: float = 1.0

    def validate(self) -> None:
        if self.kind not in ("gaussian", "linear"):
            raise ValueError(f"unknown kernel kind {self.kind!r}")
        if self.kind == "gaussian" and self.sigma <= 0:
            raise ValueError(f"sigma must be > 0, got {self.sigma}")


@dataclass
class SvmModel:
    """Support set, dual weights, labels, bias, kernel (svm.py:51-60)."""

    support_points: np.ndarray
    support_duals: np.ndarray
    support_labels: np.ndarray
    bias: float
    kernel: KernelSpec
    C: float


@dataclass
class TrainDiagnostics:
    """svm.py:171-178."""

    iterations: int
    status: Status
    primal_residual_history: np.ndarray
    dual_residual_history: np.ndarray
    duals: np.ndarray
    eq_dual: float


def _rows(X: Matrix) -> np.ndarray:
    if sp.issparse(X):
        return np.asarray(X.todense(), dtype=float)
    if isinstance(X, torch.Tensor):
        return X.detach().cpu().numpy().astype(float)
    return np.asarray(X, dtype=float)


def default_block_size(n: int) -> int:
    """svm.py:146-152."""
    if n < 30_000:
        return min(100, n)
    if n < 100_000:
        return 500
    return 1000


def default_config(n: int, block_size: Optional[int] = None, seed: int = 0, max_iters: int = 10,
                   tol_primal: float = 1e-1, tol_dual: float = 1.0, mode: Mode = Mode.RAC,
                   beta: Optional[float] = None) -> SolverConfig:
    """Loose tolerances, few sweeps, beta = 0.1 * #blocks (svm.py:155-168)."""
    s = min(block_size or default_block_size(n), n)
    p = math.ceil(n / s)
    return SolverConfig(mode=mode, block_size=s, beta_penalty=beta if beta is not None else 0.1 * p,
                        max_iters=max_iters, tol_primal=tol_primal, tol_dual=tol_dual, seed=seed)


def build_q(X: np.ndarray, y: np.ndarray, kernel: KernelSpec, device=None) -> torch.Tensor:
    """Q = y_i y_j K(x_i, x_j) on the device (N x N fp64), one DMMA SYRK + epilogue."""
    dev = _device.require_cuda(device)
    lib = _native.load()
    N, d = X.shape
    Xd = _device.upload(X, device=dev)
    yd = _device.upload(y, device=dev)
    Q = torch.empty((N, N), dtype=torch.float64, device=dev)
    kind = _native.KERNEL_LINEAR if kernel.kind == "linear" else _native.KERNEL_GAUSSIAN
    _native.check(lib.rac_svm_build_q(Xd.data_ptr(), N, d, yd.data_ptr(), kind, float(kernel.sigma),
                                      Q.data_ptr(), _device.stream_handle(device=dev)))
    torch.cuda.current_stream(dev).synchronize()
    return Q


def _bias_from_q(Q: torch.Tensor, z: np.ndarray, y: np.ndarray, C: float) -> float:
    """compute_bias (svm.py:287-322) with g = y * (Q (z on the support)) from the device Q."""
    support = z > SUPPORT_THRESHOLD
    if not np.any(support):
        raise DegenerateModelError("no support vectors; cannot recover a bias")
    lib = _native.load()
    w = torch.from_numpy(np.where(support, z, 0.0)).to(Q.device)
    qz = torch.empty(Q.shape[0], dtype=torch.float64, device=Q.device)
    _native.check(lib.rac_gemv(Q.data_ptr(), Q.shape[0], Q.shape[1], w.data_ptr(), qz.data_ptr(),
                               _device.stream_handle(device=Q.device)))
    g = y * qz.cpu().numpy()     # sum_j y_j z_j K(x_j, x_i) = y_i (Q z_sup)_i
    margin = (z > MARGIN_DELTA * C) & (z < (1.0 - MARGIN_DELTA) * C)
    if np.any(margin):
        return _bias_from_g(g[margin], np.flatnonzero(margin), z, y, C, True)
    return _bias_from_g(g, np.arange(y.size), z, y, C, False)


def _bias_from_g(g: np.ndarray, rows: np.ndarray, z: np.ndarray, y: np.ndarray, C: float, margin: bool) -> float:
    """Margin mean, else the midpoint of the interval the bound KKT conditions allow (svm.py:304-322);
    `g` holds sum_j y_j z_j K(x_j, x_i) for the samples `rows`."""
    if margin:
        return float(np.mean(y[rows] - g))
    vals = y - g
    at_upper = z >= (1.0 - MARGIN_DELTA) * C
    at_lower = ~at_upper
    lower_b = vals[(at_lower & (y > 0)) | (at_upper & (y < 0))]
    upper_b = vals[(at_lower & (y < 0)) | (at_upper & (y > 0))]
    lo = float(np.max(lower_b)) if lower_b.size else -math.inf
    hi = float(np.min(upper_b)) if upper_b.size else math.inf
    if not math.isfinite(lo):
        return hi
    if not math.isfinite(hi):
        return lo
    return (lo + hi) / 2.0


def train(X: Matrix, labels: np.ndarray, C: float, kernel: KernelSpec,
          config: Optional[SolverConfig] = None, cache_capacity: Optional[int] = None,
          return_diagnostics: bool = False, sweep_hook=None, device=None):
    """Train a classifier by sweeping the dual QP blockwise (svm.py:181-284).

    `sweep_hook(k, z, nu)` (optional, not in the reference) observes each sweep; `device`
    (not in the reference) is the CUDA device, default the current one.
    """
    kernel.validate()
    Xd = _rows(X)
    y = np.asarray(labels, dtype=float)
    n = Xd.shape[0]
    if y.size != n:
        raise ValueError(f"labels length {y.size} does not match {n} rows")
    if not np.all(np.isin(y, (-1.0, 1.0))):
        raise ValueError("labels must be -1 or +1")
    if C <= 0:
        raise ValueError(f"C must be > 0, got {C}")
    if config is None:
        config = default_config(n)
    config.validate(n)
    mode = Mode(config.mode)
    rng = np.random.default_rng(config.seed)
    dev = _device.require_cuda(device)
    with torch.cuda.device(dev):
        return _train_on(dev, Xd, y, C, kernel, config, mode, rng, return_diagnostics, sweep_hook)


def use_kernel_strips(n: int, mode: Mode, device) -> bool:
    """Kernel strips on the fly (the reference's own scheme, svm.py:96-143) when the n x n
    label-weighted kernel matrix would take more than half of the free device memory, or
    RAC_SVM_STRIPS=1; RAC_SVM_STRIPS=0 forces the resident matrix.  RP visits blocks out of
    table order and keeps the resident matrix."""
    env = os.environ.get("RAC_SVM_STRIPS")
    if env is not None:
        return env == "1" and Mode(mode) != Mode.RP
    free, _ = torch.cuda.mem_get_info(device)
    return 8.0 * n * n > 0.5 * free and Mode(mode) != Mode.RP


STRIP_BYTES = 2 << 30      # strip rows formed per batch of blocks


def _train_on(dev, Xd, y, C, kernel, config, mode, rng, return_diagnostics, sweep_hook):
    n = Xd.shape[0]
    strips = use_kernel_strips(n, mode, dev)
    Q = None if strips else build_q(Xd, y, kernel, dev)
    solver = QpSolver(n, 1, config.block_size, mode, config.beta_penalty, RIDGE_REL, device=dev)
    try:
        if strips:
            kind = _native.KERNEL_LINEAR if kernel.kind == "linear" else _native.KERNEL_GAUSSIAN
            solver.set_kernel_strips(Xd, y, kind, kernel.sigma, STRIP_BYTES)
        solver.set_problem(np.full(n, -1.0), np.zeros(n), np.full(n, float(C)),
                           A=y.reshape(1, n), b=np.zeros(1), borrowed_h=Q)
        solver.set_divergence_bar(math.inf)   # train has no divergence guard
        if mode == Mode.CYCLIC:
            solver.set_partition(np.arange(n))
        elif mode == Mode.RP:
            solver.set_partition(rng.permutation(n))
        hook = None if sweep_hook is None else (lambda k, x, yv: sweep_hook(k, x, float(yv[0])))
        it, status = drive(solver, rng, config.max_iters, config.tol_primal, config.tol_dual,
                           config.fixed_iterations, hook=hook)
        x, yv, _ = solver.state()
        hp, _, hd = (h.cpu().numpy() for h in solver.history(it))
        z = x.cpu().numpy()
        nu = float(yv.cpu().numpy()[0])
    finally:
        solver.close()
    bias = compute_bias(z, Xd, y, C, kernel, device=dev) if strips else _bias_from_q(Q, z, y, C)
    del Q
    support = z > SUPPORT_THRESHOLD
    model = SvmModel(support_points=_gather_rows(Xd, support), support_duals=z[support].copy(),
                     support_labels=y[support].copy(), bias=bias, kernel=kernel, C=C)
    if return_diagnostics:
        return model, TrainDiagnostics(iterations=it, status=status, primal_residual_history=hp,
                                       dual_residual_history=hd, duals=z, eq_dual=nu)
    return model


def _gather_rows(X: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """X[mask] as a fresh array; multi-threaded index_select (the boolean-mask copy of the
    support vectors is single-threaded numpy: ~4x slower for config 4's 80 MB)."""
    rows = np.flatnonzero(mask)
    Xc = np.ascontiguousarray(X)
    return torch.from_numpy(Xc).index_select(0, torch.from_numpy(rows)).numpy()


# ---------------------------------------------------------------- reference helpers on the device
class KernelRowCache:
    """Signature twin of svm.py:96-118.  The device forms whole strips at once
    (rac_svm_kernel_strip), so the cache is only carried through; `hits`/`misses` count
    the rows asked for."""

    def __init__(self, X: np.ndarray, kernel: KernelSpec, capacity: int):
        self.X = X
        self.kernel = kernel
        self.capacity = max(1, capacity)
        self.hits = 0
        self.misses = 0


def _strip_rows(Xd: np.ndarray, y: np.ndarray, rows: np.ndarray, kernel: KernelSpec, dev) -> torch.Tensor:
    """(len(rows) x N) label-weighted kernel strip on the device."""
    lib = _native.load()
    N, d = Xd.shape
    Xg = _device.upload(Xd, device=dev)
    yg = _device.upload(y, device=dev)
    rg = torch.from_numpy(np.asarray(rows, dtype=np.int32)).to(dev)
    out = torch.empty((rows.size, N), dtype=torch.float64, device=dev)
    kind = _native.KERNEL_LINEAR if kernel.kind == "linear" else _native.KERNEL_GAUSSIAN
    _native.check(lib.rac_svm_kernel_strip(Xg.data_ptr(), N, d, yg.data_ptr(), rg.data_ptr(), int(rows.size), kind,
                                           float(kernel.sigma), out.data_ptr(), _device.stream_handle(device=dev)))
    return out


def assemble_kernel_block(X: Matrix, y: np.ndarray, block, kernel: KernelSpec,
                          cache: Optional[KernelRowCache] = None, with_strip: bool = False, *, device=None):
    """Label-weighted kernel block Q_bb (and with `with_strip` the s x N strip Q_b.)
    straight from the data rows, on the FP64 tensor cores (svm.py:121-143)."""
    kernel.validate()
    Xd = _rows(X)
    y = np.asarray(y, dtype=float)
    idx = np.asarray(block, dtype=np.int64)
    dev = _device.require_cuda(device)
    with torch.cuda.device(dev):
        strip = _strip_rows(Xd, y, idx, kernel, dev)
        if cache is not None:
            cache.misses += int(idx.size)
        qbb = strip[:, torch.from_numpy(idx).to(dev)]
        if with_strip:
            return qbb.cpu().numpy(), strip.cpu().numpy()
        return qbb.cpu().numpy()


def kernel_eval(xi: np.ndarray, xj: np.ndarray, kernel: KernelSpec) -> float:
    """K(x_i, x_j) for one pair (svm.py:68-79); scalar host helper."""
    kernel.validate()
    xi, xj = np.asarray(xi, dtype=float), np.asarray(xj, dtype=float)
    if xi.shape != xj.shape:
        raise ValueError(f"feature dimensions differ: {xi.shape} vs {xj.shape}")
    if kernel.kind == "linear":
        return float(xi @ xj)
    return math.exp(-float(np.sum((xi - xj) ** 2)) / (2.0 * kernel.sigma ** 2))


def compute_bias(duals: np.ndarray, X: Matrix, labels: np.ndarray, C: float, kernel: KernelSpec, *,
                 device=None) -> float:
    """Bias from the margin support vectors (svm.py:287-322).  g_i = sum_j y_j z_j K(x_j, x_i)
    = y_i (Q z_sup)_i is formed from device kernel strips of the needed rows (chunks of at
    most 2048 rows), then the reference's margin mean / bracket midpoint."""
    Xd = _rows(X)
    y = np.asarray(labels, dtype=float)
    z = np.asarray(duals, dtype=float)
    support = z > SUPPORT_THRESHOLD
    if not np.any(support):
        raise DegenerateModelError("no support vectors; cannot recover a bias")
    margin = (z > MARGIN_DELTA * C) & (z < (1.0 - MARGIN_DELTA) * C)
    need = np.flatnonzero(margin) if np.any(margin) else np.arange(y.size)
    dev = _device.require_cuda(device)
    lib = _native.load()
    with torch.cuda.device(dev):
        w = torch.from_numpy(np.where(support, z, 0.0)).to(dev)
        qz = np.empty(need.size)
        for c0 in range(0, need.size, 2048):
            rows = need[c0:c0 + 2048]
            strip = _strip_rows(Xd, y, rows, kernel, dev)
            out = torch.empty(rows.size, dtype=torch.float64, device=dev)
            _native.check(lib.rac_gemv(strip.data_ptr(), rows.size, y.size, w.data_ptr(), out.data_ptr(),
                                       _device.stream_handle(device=dev)))
            qz[c0:c0 + rows.size] = out.cpu().numpy()
    g = y[need] * qz
    return _bias_from_g(g, need, z, y, C, bool(np.any(margin)))


# ---------------------------------------------------------------- host post-processing
def kernel_cross(Xa: np.ndarray, Xb: np.ndarray, kernel: KernelSpec) -> np.ndarray:
    """K between rows of Xa and Xb (svm.py:82-93); post-processing helper."""
    kernel.validate()
    Xa, Xb = np.asarray(Xa, dtype=float), np.asarray(Xb, dtype=float)
    if kernel.kind == "linear":
        return Xa @ Xb.T
    d2 = np.maximum(np.sum(Xa * Xa, axis=1)[:, None] + np.sum(Xb * Xb, axis=1)[None, :]
                    - 2.0 * (Xa @ Xb.T), 0.0)
    return np.exp(-d2 / (2.0 * kernel.sigma ** 2))


def decision_values(model: SvmModel, X_query: Matrix) -> np.ndarray:
    """f(x) = sum_i y_i z_i K(x_i, x) + b (svm.py:325-333)."""
    Xq = _rows(X_query)
    if Xq.shape[1] != model.support_points.shape[1]:
        raise ValueError(f"query has {Xq.shape[1]} features, model expects "
                         f"{model.support_points.shape[1]}")
    k = kernel_cross(Xq, model.support_points, model.kernel)
    return k @ (model.support_labels * model.support_duals) + model.bias


def predict(model: SvmModel, X_query: Matrix) -> np.ndarray:
    f = decision_values(model, X_query)
    return np.where(f >= 0.0, 1.0, -1.0)


def accuracy(model: SvmModel, X_test: Matrix, y_test: np.ndarray) -> float:
    y_test = np.asarray(y_test, dtype=float)
    return float(np.mean(predict(model, X_test) == y_test)) * 100.0
