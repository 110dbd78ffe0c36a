"""Elastic-net / LASSO / ridge by RAC block sweeps on one B200.

Drop-in for racml.elastic_net (elastic_net.py:51-232): same ElasticNetSpec,
same ElasticNetModel fields, same fit(X, y, spec) signature, validation
messages and BlockDefinitenessError.  The sweep itself runs in the native
sm_100a engine (`rac_en_*`, include/rac_b200.h); the host only draws the
reference's PCG64 permutations and streams them to the device.
"""

from __future__ import annotations

import collections
import itertools
import math
import os
import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.sparse as sp
import torch

from . import _device, _native
from .engine import BlockDefinitenessError
from .problems import Matrix, Mode

AUTO_GAMMA_DENSITY = 0.005   # elastic_net.py:48


@dataclass(frozen=True)
class ElasticNetSpec:
    """Regression hyperparameters and sweep settings (elastic_net.py:51-76)."""

    lam: float
    alpha: float
    gamma: Optional[float] = None
    block_size: int = 100
    iters: int = 10
    mode: Mode = Mode.RAC
    seed: int = 0
    tol: Optional[float] = None

    def validate(self) -> None:
        if self.lam < 0:
            raise ValueError(f"lam must be >= 0, got {self.lam}")
        if not (0.0 <= self.alpha <= 1.0):
            raise ValueError(f"alpha must be in [0, 1], got {self.alpha}")
        if self.gamma is not None and self.gamma <= 0:
            raise ValueError(f"gamma must be > 0, got {self.gamma}")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        if self.iters < 1:
            raise ValueError("iters must be >= 1")
        if Mode(self.mode) not in (Mode.RAC, Mode.RP):
            raise ValueError(f"mode must be rac or rp, got {self.mode}")


@dataclass
class ElasticNetModel:
    """Fitted coefficients and splitting state (elastic_net.py:79-89).

    Extra (drop-in compatible) fields: per-sweep ||beta - z||_1 history and
    gamma * ||z_k - z_{k-1}||_inf (a dual residual the reference does not
    define; reported, never used for stopping).
    """

    beta: np.ndarray
    z: np.ndarray
    xi: np.ndarray
    spec: ElasticNetSpec
    gamma: float
    iterations: int
    residual: float
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    dual_residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))


def density(X) -> float:
    """Stored-nonzero fraction (data_io.py:213-220)."""
    total = X.shape[0] * X.shape[1]
    if total == 0:
        return 0.0
    if sp.issparse(X):
        return X.count_nonzero() / total
    if isinstance(X, torch.Tensor):
        return float(torch.count_nonzero(X).item()) / total
    return float(np.count_nonzero(X)) / total


def resolve_gamma(spec: ElasticNetSpec, X) -> float:
    """elastic_net.py:92-99."""
    if spec.gamma is not None:
        return spec.gamma
    if spec.lam == 0.0:
        return 1.0
    return 0.1 * spec.lam if density(X) >= AUTO_GAMMA_DENSITY else spec.lam


def soft_threshold(a, b):
    """Negated shrinkage -sign(a) max(|a| - b, 0) (elastic_net.py:102-115); API twin."""
    a = np.asarray(a, dtype=float)
    if np.any(np.asarray(b) < 0):
        raise ValueError("threshold b must be >= 0")
    out = -np.sign(a) * np.maximum(np.abs(a) - b, 0.0) + 0.0
    return float(out) if out.ndim == 0 else out


def z_update(beta_i, xi_i, gamma: float, lam: float, alpha: float):
    """Closed-form z minimizer (elastic_net.py:118-131).

    torch CUDA tensors run the device kernel (`rac_z_prox`, the same code the
    fused sweep uses); numpy inputs keep the reference's host semantics.
    """
    if gamma <= 0:
        raise ValueError(f"gamma must be > 0, got {gamma}")
    denom = (1.0 - alpha) * lam + gamma
    if isinstance(beta_i, torch.Tensor) and beta_i.is_cuda:
        b = beta_i.contiguous().to(torch.float64)
        x = torch.as_tensor(xi_i, device=b.device, dtype=torch.float64).contiguous()
        z = torch.empty_like(b)
        lib = _native.load()
        _native.check(lib.rac_z_prox(b.data_ptr(), x.data_ptr(), b.numel(), gamma, lam * alpha,
                                     denom, z.data_ptr(), _device.stream_handle()))
        return z
    a = np.asarray(xi_i, dtype=float) - gamma * np.asarray(beta_i, dtype=float)
    out = soft_threshold(a, lam * alpha) / denom
    return float(out) if np.ndim(out) == 0 else out


def objective(X: Matrix, y: np.ndarray, beta: np.ndarray, lam: float, alpha: float) -> float:
    """(1/2n)||y - X beta||^2 + lam(alpha||beta||_1 + (1-alpha)/2||beta||^2) (elastic_net.py:134-141)."""
    n = X.shape[0]
    r = X @ beta - y
    penalty = lam * (alpha * np.sum(np.abs(beta)) + 0.5 * (1.0 - alpha) * float(beta @ beta))
    return 0.5 * float(r @ r) / n + penalty


class EnSolver:
    """One native elastic-net sweep context (rac_en_ctx) on the current stream."""

    def __init__(self, m: int, n: int, block_size: int, mode: Mode, lam: float, alpha: float,
                 gamma: float, device=None):
        self.dev = _device.require_cuda(device)
        self.lib = _native.load()
        self.m, self.n = int(m), int(n)
        self.s = min(int(block_size), self.n)
        self.p = -(-self.n // self.s)
        self.mode = Mode(mode)
        self.stream = _device.stream_handle(device=self.dev)
        h = _native._p()
        with torch.cuda.device(self.dev):    # the context allocates and launches on this device
            _native.check(self.lib.rac_en_create(
                h, self.m, self.n, self.s,
                _native.MODE_RP if self.mode == Mode.RP else _native.MODE_RAC,
                float(lam), float(alpha), float(gamma), self.stream))
        self.h = h
        self._keep = []
        self.gram_mode = "blocks"

    def set_gram_mode(self, mode: str) -> None:
        """'blocks': per-sweep X_b'X_b from X (the reference's own recompute);
        'covariance': G = X'X/m once, chain on G (RAC_GRAM_COVARIANCE).
        Selecting 'covariance' again re-forms G on the next run."""
        code = {"blocks": _native.GRAM_BLOCKS, "covariance": _native.GRAM_COVARIANCE}[mode]
        _native.check(self.lib.rac_en_set_gram_mode(self.h, code))
        self.gram_mode = mode

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.rac_en_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_data(self, X, y) -> None:
        """X: numpy (C or F order) / scipy sparse / torch tensor; y: length m."""
        layout = _native.LAYOUT_ROW_MAJOR
        if sp.issparse(X):
            self._set_data_csc(X, y)
            return
        if isinstance(X, torch.Tensor):
            Xd = X.to(self.dev, torch.float64)
            if not Xd.is_contiguous() and Xd.t().is_contiguous():
                layout = _native.LAYOUT_COL_MAJOR
            else:
                Xd = Xd.contiguous()
        else:
            X = np.asarray(X, dtype=float)
            if X.flags.f_contiguous and not X.flags.c_contiguous:
                Xd = _device.upload(X.T, device=self.dev)   # (n, m) C-order == column-major X
                layout = _native.LAYOUT_COL_MAJOR
            elif X.nbytes > 2 * _device.ROW_CHUNK_BYTES and self.m >= 64:
                self._set_data_streamed(X, y)
                return
            else:
                Xd = _device.upload(X, device=self.dev)
        yd = _device.upload(y, device=self.dev)
        _native.check(self.lib.rac_en_set_data(self.h, Xd.data_ptr(), layout, yd.data_ptr()))
        self._keep = [Xd, yd]   # alive until the stream consumed them

    def _set_data_csc(self, X, y) -> None:
        """Sparse X: upload the CSC arrays (nnz-sized) and expand on the device (rac_en_set_data_csc)."""
        A = sp.csc_matrix(X, dtype=np.float64, copy=True)
        A.sum_duplicates()          # canonical: sorted rows, duplicates summed (what todense gives)
        A.sort_indices()
        if A.nnz >= 2 ** 31 or self.m >= 2 ** 31:
            raise ValueError("sparse X too large for 32-bit row indices")
        ip = _device.upload(A.indptr.astype(np.int64), dtype=torch.int64, device=self.dev)
        rows = vals = None
        if A.nnz:
            rows = torch.from_numpy(A.indices.astype(np.int32)).to(self.dev)
            vals = _device.upload(A.data, device=self.dev)
        yd = _device.upload(y, device=self.dev)
        _native.check(self.lib.rac_en_set_data_csc(self.h, ip.data_ptr(), _device.ptr(rows), _device.ptr(vals),
                                                   yd.data_ptr()))
        self._keep = [ip, rows, vals, yd]

    def _set_data_streamed(self, X: np.ndarray, y) -> None:
        """Host X in row chunks: the transfer of chunk k+1 overlaps the device
        transpose (and, in covariance mode, G += X_k'X_k) of chunk k."""
        yd = _device.upload(y, device=self.dev)
        last = {}

        def consume(r0, rows, chunk):
            done = r0 + rows == self.m
            _native.check(self.lib.rac_en_set_data_rows(self.h, chunk.data_ptr(), r0, rows,
                                                        yd.data_ptr() if done else None))
            last["keep"] = chunk

        _device.stream_rows(X, 32, consume, device=self.dev)
        self._keep = [yd, last.get("keep")]

    def reset(self, lam: float, alpha: float, gamma: float) -> None:
        """Re-arm for a new fit of the same shape (rac_en_reset): iterates, history and
        failure state cleared; data (and partition / G) must be set again."""
        _native.check(self.lib.rac_en_reset(self.h, float(lam), float(alpha), float(gamma)))
        self._keep = []

    def results(self, count: int):
        """beta, z, xi and the first `count` residual histories in ONE device->host copy."""
        n = self.n
        buf = torch.empty(3 * n + 2 * max(count, 1), dtype=torch.float64, device=self.dev)
        _native.check(self.lib.rac_en_get(self.h, buf.data_ptr(), buf[n:].data_ptr(), buf[2 * n:].data_ptr(), None))
        if count > 0:
            _native.check(self.lib.rac_en_history(self.h, buf[3 * n:].data_ptr(), buf[3 * n + count:].data_ptr(),
                                                  count))
        h = buf.cpu().numpy()
        return h[:n], h[n:2 * n], h[2 * n:3 * n], h[3 * n:3 * n + count], h[3 * n + count:3 * n + 2 * count]

    def set_partition(self, perm_dev: torch.Tensor) -> None:
        _native.check(self.lib.rac_en_set_partition(self.h, perm_dev.data_ptr()))

    def run(self, perms_dev: torch.Tensor, tol: Optional[float]) -> None:
        count = perms_dev.shape[0]
        _native.check(self.lib.rac_en_run(self.h, perms_dev.data_ptr(), count,
                                          -1.0 if tol is None else float(tol)))

    def progress(self):
        it, conv, fb = _native._i32(), _native._i32(), _native._i32()
        res = _native._f64()
        _native.check(self.lib.rac_en_progress(self.h, it, conv, res, fb))
        return it.value, bool(conv.value), res.value, fb.value

    def poll(self, lag: int = 1):
        """(iterations, converged, failed_block) after the run `lag` runs before the latest,
        waiting only for that run (rac_en_poll)."""
        it, conv, fb = _native._i32(), _native._i32(), _native._i32()
        _native.check(self.lib.rac_en_poll(self.h, int(lag), it, conv, fb))
        return it.value, bool(conv.value), fb.value

    def state(self):
        b = torch.empty(self.n, dtype=torch.float64, device=self.dev)
        z, xi = torch.empty_like(b), torch.empty_like(b)
        _native.check(self.lib.rac_en_get(self.h, b.data_ptr(), z.data_ptr(), xi.data_ptr(), None))
        return b, z, xi

    def history(self, count: int):
        hp = torch.empty(max(count, 1), dtype=torch.float64, device=self.dev)
        hd = torch.empty_like(hp)
        _native.check(self.lib.rac_en_history(self.h, hp.data_ptr(), hd.data_ptr(), count))
        return hp[:count], hd[:count]


COV_MAX_N = 20000

# fit() reuses native contexts of the same shape (rac_en_reset) instead of creating and
# destroying one per call: streams, events, plans and pool buffers stay; each fit holds
# its context exclusively.  At most _POOL_MAX idle contexts and about _POOL_BYTES of
# their device memory are kept (least recently used closed first); release_pool() closes
# them all and returns the memory to the driver.
_POOL: "collections.OrderedDict" = collections.OrderedDict()   # (key, serial) -> solver
_POOL_LOCK = threading.Lock()
_POOL_MAX = 4
_POOL_BYTES = int(os.environ.get("RAC_POOL_BYTES", str(24 << 30)))
_POOL_SERIAL = itertools.count()


def _ctx_bytes(key) -> int:
    """Rough device footprint of a pooled context: X (column-major), its int8 digit slices,
    G (covariance mode) and the per-sweep block inverses, double-buffered."""
    m, n, s = key[0], key[1], key[2]
    p = -(-n // s)
    return 16 * m * n + (8 * n * n if n <= COV_MAX_N else 0) + 16 * p * s * s


def release_pool() -> None:
    """Close every idle pooled fit context and trim the native memory pool (e.g. before a
    large allocation by other code)."""
    with _POOL_LOCK:
        idle = list(_POOL.values())
        _POOL.clear()
    for sv in idle:
        sv.close()
    if torch.cuda.is_available():
        _native.check(_native.load().rac_trim_pool(0))


def _acquire_solver(m, n, block_size, mode, lam, alpha, gamma, device):
    # RAC_* environment switches select native variants when a context is created / planned
    env = tuple(sorted((k, v) for k, v in os.environ.items() if k.startswith("RAC_")))
    key = (m, n, min(int(block_size), n), Mode(mode), device, _device.stream_handle(device=device), env)
    solver = None
    with _POOL_LOCK:
        for pk in reversed(_POOL):
            if pk[0] == key:
                solver = _POOL.pop(pk)
                break
    if solver is not None:
        solver.reset(lam, alpha, gamma)
        return key, solver
    return key, EnSolver(m, n, block_size, mode, lam, alpha, gamma, device=device)


def _release_solver(key, solver, ok: bool) -> None:
    evicted = []
    if ok:
        with _POOL_LOCK:
            _POOL[(key, next(_POOL_SERIAL))] = solver
            while len(_POOL) > _POOL_MAX or (len(_POOL) > 1 and
                                            sum(_ctx_bytes(k[0]) for k in _POOL) > _POOL_BYTES):
                evicted.append(_POOL.popitem(last=False)[1])
    else:
        evicted.append(solver)
    for sv in evicted:
        sv.close()


def choose_gram_mode(m: int, n: int, block_size: int, iters: int) -> str:
    """Covariance mode pays when G (n x n) is small next to X and the fit runs
    enough sweeps to amortise forming it: m n^2 / 2 flops once versus
    m n (s + 1) per sweep for the block Grams, i.e. iters >~ p / 2."""
    s = max(1, min(int(block_size), n))
    p = -(-n // s)
    if n > COV_MAX_N or n > 2 * m:
        return "blocks"
    return "covariance" if iters >= max(2, (p + 1) // 2) else "blocks"


def fit(X: Matrix, y: np.ndarray, spec: ElasticNetSpec, *, sweep_hook=None,
        batch: int = 16, device=None, gram_mode: str = "auto") -> ElasticNetModel:
    """Randomized block-sweep fit of the elastic-net objective (elastic_net.py:150-232).

    Same arguments, results and errors as the reference.  `sweep_hook(k, beta,
    z, xi)` (optional, not in the reference) observes every sweep; it forces a
    device->host copy per sweep and is meant for parity capture.  `gram_mode`
    (optional, not in the reference): "blocks", "covariance" or "auto"
    (choose_gram_mode); both give the reference's iterates to rounding.
    """
    spec.validate()
    m, n = X.shape
    if m < 1 or n < 1:
        raise ValueError("X must be non-empty")
    if isinstance(y, torch.Tensor):
        y = y.detach().cpu().numpy()
    y = np.asarray(y, dtype=float)
    if y.size != m:
        raise ValueError(f"y has length {y.size}, expected {m}")
    gamma = resolve_gamma(spec, X)
    dev = _device.require_cuda(device)
    with torch.cuda.device(dev):     # the pooled context, its stream and uploads live on `dev`
        return _fit_on(dev.index, X, y, spec, m, n, gamma, sweep_hook, batch, gram_mode)


def _fit_on(device: int, X, y, spec: ElasticNetSpec, m: int, n: int, gamma: float, sweep_hook, batch: int,
            gram_mode: str) -> ElasticNetModel:
    mode = Mode(spec.mode)
    rng = np.random.default_rng(spec.seed)
    key, solver = _acquire_solver(m, n, spec.block_size, mode, spec.lam, spec.alpha, gamma, device)
    ok = False
    try:
        gm = choose_gram_mode(m, n, spec.block_size, spec.iters) if gram_mode == "auto" else gram_mode
        if gm == "covariance":
            try:
                solver.set_gram_mode("covariance")
            except _native.NativeError as e:
                if e.code != _native.RAC_ERR_UNSUPPORTED or gram_mode != "auto":
                    raise
                solver.set_gram_mode("blocks")
        else:
            solver.set_gram_mode("blocks")
        solver.set_data(X, y)
        if mode == Mode.RP:
            solver.set_partition(_device.PermutationFeeder(rng, n, solver.dev).draw(1))
            feeder = _device.PermutationFeeder(rng, solver.p, solver.dev)
        else:
            feeder = _device.PermutationFeeder(rng, n, solver.dev)
        step = 1 if sweep_hook is not None else max(1, int(batch))
        # the first batch is drawn before any sweep can start: keep its host time (~1 us per 100
        # coordinates per sweep) small; later batches are drawn while the device runs
        first = max(1, min(step, 200_000 // max(1, feeder.size)))
        done = 0
        iterations, converged, failed = 0, False, -1
        if sweep_hook is None and spec.tol is not None and spec.iters > 0:
            # with a tolerance: batch k+1 is enqueued before batch k's status is read (a
            # non-blocking poll of the run before the latest), so no host round trip
            # separates the batches; launches after convergence are no-ops on the device
            solver.run(feeder.draw(min(first, spec.iters)), spec.tol)
            done = min(first, spec.iters)
            while True:
                lag = 0
                if done < spec.iters:
                    k = min(step, spec.iters - done)
                    solver.run(feeder.draw(k), spec.tol)
                    done += k
                    lag = 1
                _, conv, failed = solver.poll(lag)
                if failed >= 0 or conv or lag == 0:
                    break
            done = spec.iters          # the final progress() below reports the true state
        perms = feeder.draw(min(first, spec.iters)) if done < spec.iters else None
        while done < spec.iters:
            k = perms.shape[0]
            solver.run(perms, spec.tol)
            done += k
            # the next batch's permutations are drawn (host PCG64, same stream order) while
            # the device runs this one; a batch drawn past convergence is simply dropped
            perms = feeder.draw(min(step, spec.iters - done)) if done < spec.iters else None
            if sweep_hook is not None or spec.tol is not None or done >= spec.iters:
                iterations, converged, _, failed = solver.progress()
                if failed >= 0:
                    ok = True   # the context itself is sound; the next fit resets it
                    raise BlockDefinitenessError(
                        "sub-block Gram matrix plus gamma*I is not positive definite; the "
                        "sub-block positive-definiteness requirement is violated")
                if sweep_hook is not None and iterations == done:
                    b, z, xi = solver.state()
                    sweep_hook(iterations, b.cpu().numpy(), z.cpu().numpy(), xi.cpu().numpy())
                if converged:
                    break
        iterations, converged, residual, failed = solver.progress()
        if failed >= 0:
            ok = True   # the context itself is sound; the next fit resets it
            raise BlockDefinitenessError(
                "sub-block Gram matrix plus gamma*I is not positive definite; the "
                "sub-block positive-definiteness requirement is violated")
        b, z, xi, hp, hd = solver.results(iterations)
        ok = True
        return ElasticNetModel(beta=b.copy(), z=z.copy(), xi=xi.copy(),
                               spec=spec, gamma=gamma, iterations=iterations,
                               residual=residual if iterations else math.inf,
                               residual_history=hp.copy(), dual_residual_history=hd.copy())
    finally:
        _release_solver(key, solver, ok)


from .consensus import consensus_fit  # noqa: E402  (the consensus baseline, elastic_net.py:252-316)
