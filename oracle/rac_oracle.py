"""CPU oracle for the RAC-MBADMM sweep — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy/scipy restatement of the reference algorithm
(`racml` 0.1.0 under /root/reference/pkg/src/racml).  It exists so that

  * `tests/` can check the CUDA path against a CPU answer on the GPU box
    (where /root/reference does not exist), and
  * `bench.py --impl reference` / the `cpu_baseline` leg can time the
    reference's CPU algorithm on the GPU box's host cores ("port").

Nothing in the product package (`paper_1907_01995_b200/`) may import it.

Parity pinning: `tests/golden/make_golden.py` runs the *real* reference in
the build container and stores its per-sweep iterates as fixtures;
`tests/test_oracle_golden.py` checks this restatement against them
(bit-exact for block indices, <=1e-13 relative for iterates).

Each function cites the reference lines it restates.  The numpy operation
order follows the reference so that results agree to rounding.
"""

from __future__ import annotations

import math
from typing import Callable, Optional

import numpy as np
import scipy.linalg

RAC, RP, CYCLIC = "rac", "rp", "cyclic"

# engine.py:34-39
DIVERGENCE_FACTOR = 1e8
ACTIVE_SET_PASS_FACTOR = 10
PG_TOL = 1e-10
# svm.py:25-26
SUPPORT_THRESHOLD = 1e-8
MARGIN_DELTA = 1e-6
# elastic_net.py:48
AUTO_GAMMA_DENSITY = 0.005


class NotPositiveDefinite(ArithmeticError):
    """Oracle twin of racml.engine.BlockDefinitenessError."""


# ---------------------------------------------------------------------------
# block assembly  (problems.py:234-243, engine.py:318-319)
# ---------------------------------------------------------------------------

def sorted_chunks(perm: np.ndarray, s: int) -> list[np.ndarray]:
    """Cut `perm` into consecutive chunks of `s`, each sorted ascending."""
    perm = np.asarray(perm)
    return [np.sort(perm[k:k + s]).astype(np.int64)
            for k in range(0, perm.size, s)]


def sweep_orders(mode: str, rng: np.random.Generator, n: int, s: int):
    """Generator of per-sweep block lists in the reference's RNG call order.

    RAC: one rng.permutation(n) per sweep (elastic_net.py:194-195,
    svm.py:230-231, engine.py:370-371).  RP: one permutation(n) up front,
    then permutation(p) per sweep (elastic_net.py:187-198, engine.py:350-373).
    CYCLIC: consecutive blocks in fixed order (engine.py:348-349).
    """
    if mode == RAC:
        while True:
            yield sorted_chunks(rng.permutation(n), s)
    elif mode == RP:
        fixed = sorted_chunks(rng.permutation(n), s)
        while True:
            yield [fixed[i] for i in rng.permutation(len(fixed))]
    elif mode == CYCLIC:
        fixed = sorted_chunks(np.arange(n), s)
        while True:
            yield fixed
    else:
        raise ValueError(f"unknown mode {mode!r}")


# ---------------------------------------------------------------------------
# elastic net  (elastic_net.py:92-232)
# ---------------------------------------------------------------------------

def density(X) -> float:
    """data_io.py:213-220."""
    total = X.shape[0] * X.shape[1]
    if total == 0:
        return 0.0
    if hasattr(X, "count_nonzero") and not isinstance(X, np.ndarray):
        return X.count_nonzero() / total
    return float(np.count_nonzero(X)) / total


def auto_gamma(lam: float, gamma: Optional[float], X) -> float:
    """elastic_net.py:92-99."""
    if gamma is not None:
        return gamma
    if lam == 0.0:
        return 1.0
    return 0.1 * lam if density(X) >= AUTO_GAMMA_DENSITY else lam


def neg_shrink(a, b):
    """elastic_net.py:102-115: -sign(a)*max(|a|-b, 0), with -0 mapped to +0."""
    a = np.asarray(a, dtype=float)
    return -np.sign(a) * np.maximum(np.abs(a) - b, 0.0) + 0.0


def z_prox(beta, xi, gamma: float, lam: float, alpha: float):
    """elastic_net.py:118-131."""
    a = np.asarray(xi, dtype=float) - gamma * np.asarray(beta, dtype=float)
    return neg_shrink(a, lam * alpha) / ((1.0 - alpha) * lam + gamma)


def en_objective(X, y, beta, lam: float, alpha: float) -> float:
    """elastic_net.py:134-141."""
    res = X @ beta - y
    pen = lam * (alpha * np.sum(np.abs(beta)) + 0.5 * (1.0 - alpha) * float(beta @ beta))
    return 0.5 * float(res @ res) / X.shape[0] + pen


def _dense_cols(X, idx):
    if isinstance(X, np.ndarray):
        return X[:, idx]
    return np.asarray(X[:, idx].todense(), dtype=float)


def en_fit(X, y, lam: float, alpha: float, gamma: Optional[float] = None,
           block_size: int = 100, iters: int = 10, mode: str = RAC,
           seed: int = 0, tol: Optional[float] = None,
           on_sweep: Optional[Callable] = None) -> dict:
    """elastic_net.py:150-232 (fit).

    `on_sweep(k, blocks, beta, z, xi)` observes sweep k (1-based) after the
    dual step; `blocks` is the list of block index arrays in visit order.
    """
    m, n = X.shape
    y = np.asarray(y, dtype=float)
    g = auto_gamma(lam, gamma, X)
    rng = np.random.default_rng(seed)
    s = min(block_size, n)
    c = np.asarray(-(X.T @ y) / m, dtype=float).ravel()
    beta, z, xi = np.zeros(n), np.zeros(n), np.zeros(n)
    r = np.zeros(m)
    cache_chol = mode == RP and density(X) >= AUTO_GAMMA_DENSITY
    factors: dict = {}
    orders = sweep_orders(mode, rng, n, s)
    done, resid = 0, math.inf
    for k in range(iters):
        blocks = next(orders)
        for idx in blocks:
            Xb = _dense_cols(X, idx)
            bb = beta[idx]
            cross = Xb.T @ (r - Xb @ bb) / m
            rhs = -(c[idx] + cross - xi[idx] - g * z[idx])
            key = idx.tobytes() if cache_chol else None
            L = factors.get(key) if key is not None else None
            if L is None:
                G = (Xb.T @ Xb) / m
                G[np.diag_indices_from(G)] += g
                try:
                    L = np.linalg.cholesky(G)
                except np.linalg.LinAlgError as exc:
                    raise NotPositiveDefinite("block Gram + gamma*I not PD") from exc
                if key is not None:
                    factors[key] = L
            nb = scipy.linalg.cho_solve((L, True), rhs)
            r += Xb @ (nb - bb)
            beta[idx] = nb
        z = z_prox(beta, xi, g, lam, alpha)
        xi = xi - g * (beta - z)
        done += 1
        resid = float(np.sum(np.abs(beta - z)))
        if on_sweep is not None:
            on_sweep(done, blocks, beta, z, xi)
        if tol is not None and resid <= tol:
            break
    return dict(beta=beta, z=z, xi=xi, gamma=g, iterations=done, residual=resid)


# ---------------------------------------------------------------------------
# exact box-QP block minimizer  (engine.py:160-245)
# ---------------------------------------------------------------------------

def _chol(M):
    try:
        return np.linalg.cholesky(M)
    except np.linalg.LinAlgError as exc:
        raise NotPositiveDefinite("block matrix not positive definite") from exc


def _csolve(L, r):
    return scipy.linalg.cho_solve((L, True), r, check_finite=False)


def _pg_fallback(M, r, lo, hi, x0):
    """engine.py:175-186."""
    step = 1.0 / max(np.linalg.eigvalsh(M)[-1], 1e-12)
    x = np.clip(x0, lo, hi)
    for _ in range(200000):
        nxt = np.clip(x - step * (M @ x - r), lo, hi)
        if np.max(np.abs(nxt - x)) <= PG_TOL * step:
            return nxt
        x = nxt
    return x


def box_block_min(M, r, lo, hi, L=None, stats: Optional[dict] = None):
    """Exact minimizer of 1/2 x'Mx - r'x over [lo, hi] (engine.py:189-245)."""
    s = r.size
    if L is None:
        L = _chol(M)
    x = _csolve(L, r)
    bounded = bool(np.any(np.isfinite(lo)) or np.any(np.isfinite(hi)))
    if not bounded or (np.all(x >= lo) and np.all(x <= hi)):
        return x
    if stats is not None:
        stats["active"] = stats.get("active", 0) + 1
    x = np.clip(x, lo, hi)
    low = x <= lo
    high = x >= hi
    for _ in range(ACTIVE_SET_PASS_FACTOR * s):
        for _ in range(s + 1):
            free = ~(low | high)
            x = np.where(low, lo, np.where(high, hi, x))
            if not free.any():
                break
            F = np.flatnonzero(free)
            B = np.flatnonzero(~free)
            rr = r[F]
            if B.size:
                rr = rr - M[np.ix_(F, B)] @ x[B]
            if stats is not None:
                stats["refactor"] = stats.get("refactor", 0) + 1
            xf = _csolve(_chol(M[np.ix_(F, F)]), rr)
            vlo = xf < lo[F]
            vhi = xf > hi[F]
            x[F] = np.clip(xf, lo[F], hi[F])
            if not (vlo.any() or vhi.any()):
                break
            low[F[vlo]] = True
            high[F[vhi]] = True
        grad = M @ x - r
        scale = max(1.0, float(np.max(np.abs(grad))))
        bad_lo = low & (grad < -1e-14 * scale)
        bad_hi = high & (grad > 1e-14 * scale)
        if not (bad_lo.any() or bad_hi.any()):
            return x
        score = np.where(bad_lo, -grad, 0.0) + np.where(bad_hi, grad, 0.0)
        w = int(np.argmax(score))
        low[w] = False
        high[w] = False
    if stats is not None:
        stats["pg"] = stats.get("pg", 0) + 1
    return _pg_fallback(M, r, lo, hi, x)


# ---------------------------------------------------------------------------
# SVM dual  (svm.py:82-284)
# ---------------------------------------------------------------------------

def kernel_matrix(Xa, Xb, kind: str, sigma: float = 1.0):
    """svm.py:82-93."""
    if kind == "linear":
        return Xa @ Xb.T
    sa = np.sum(Xa * Xa, axis=1)[:, None]
    sb = np.sum(Xb * Xb, axis=1)[None, :]
    d2 = np.maximum(sa + sb - 2.0 * (Xa @ Xb.T), 0.0)
    return np.exp(-d2 / (2.0 * sigma ** 2))


def svm_train(X, labels, C: float, kind: str = "linear", sigma: float = 1.0,
              block_size: int = 100, beta: float = 1.0, max_iters: int = 10,
              tol_primal: float = 1e-6, tol_dual: float = 1e-6, seed: int = 0,
              mode: str = RAC, fixed_iterations: bool = False,
              on_sweep: Optional[Callable] = None, stats: Optional[dict] = None) -> dict:
    """svm.py:181-268 (train, without the bias/model packing).

    Kernel rows are computed per block from X exactly as the reference's
    row cache does (one `kernel_matrix(X[i:i+1], X)` per row, svm.py:114).
    `on_sweep(k, blocks, z, nu, primal, dual)` observes each sweep.
    """
    X = np.asarray(X, dtype=float)
    y = np.asarray(labels, dtype=float)
    n = X.shape[0]
    s = block_size
    rng = np.random.default_rng(seed)
    z = np.zeros(n)
    nu = 0.0
    qz = np.zeros(n)
    t = 0.0
    zeros = np.zeros(s)
    orders = sweep_orders(mode, rng, n, s)
    primal_h, dual_h = [], []
    status = "max_iters"
    sweeps = 0
    for _ in range(max_iters):
        blocks = next(orders)
        for idx in blocks:
            raw = np.stack([kernel_matrix(X[i:i + 1], X, kind, sigma)[0] for i in idx])
            strip = (y[idx][:, None] * raw) * y[None, :]
            qbb = strip[:, idx]
            yb = y[idx]
            M = qbb + beta * np.outer(yb, yb)
            M[np.diag_indices_from(M)] += 1e-9 * float(np.max(np.diag(M)))
            cross = qz[idx] - qbb @ z[idx]
            eq_rest = t - float(yb @ z[idx])
            rhs = -(-1.0 + cross - nu * yb + beta * yb * eq_rest)
            nz = box_block_min(M, rhs, zeros[:idx.size], np.full(idx.size, C), stats=stats)
            d = nz - z[idx]
            qz += strip.T @ d
            t += float(yb @ d)
            z[idx] = nz
        nu -= beta * t
        sweeps += 1
        primal = abs(t)
        grad = qz - 1.0 - nu * y
        dual = float(np.max(np.abs(np.clip(z - grad, 0.0, C) - z)))
        primal_h.append(primal)
        dual_h.append(dual)
        if on_sweep is not None:
            on_sweep(sweeps, blocks, z, nu, primal, dual)
        if not fixed_iterations and primal <= tol_primal and dual <= tol_dual:
            status = "converged"
            break
    return dict(z=z, nu=nu, qz=qz, iterations=sweeps, status=status,
                primal_history=np.asarray(primal_h), dual_history=np.asarray(dual_h))


def svm_bias(z, X, labels, C: float, kind: str = "linear", sigma: float = 1.0) -> float:
    """svm.py:287-322 (compute_bias)."""
    X = np.asarray(X, dtype=float)
    y = np.asarray(labels, dtype=float)
    sup = z > SUPPORT_THRESHOLD
    if not np.any(sup):
        raise ArithmeticError("no support vectors")
    margin = (z > MARGIN_DELTA * C) & (z < (1.0 - MARGIN_DELTA) * C)
    coef = y[sup] * z[sup]
    if np.any(margin):
        g = kernel_matrix(X[margin], X[sup], kind, sigma) @ coef
        return float(np.mean(y[margin] - g))
    g = kernel_matrix(X, X[sup], kind, sigma) @ coef
    vals = y - g
    up = z >= (1.0 - MARGIN_DELTA) * C
    dn = ~up
    lb = vals[(dn & (y > 0)) | (up & (y < 0))]
    ub = vals[(dn & (y < 0)) | (up & (y > 0))]
    lo = float(np.max(lb)) if lb.size else -math.inf
    hi = float(np.min(ub)) if ub.size else math.inf
    if not math.isfinite(lo):
        return hi
    if not math.isfinite(hi):
        return lo
    return (lo + hi) / 2.0


def svm_dual_objective(Q, z) -> float:
    """1/2 z'Qz - 1'z (test_svm.py:173)."""
    return float(0.5 * z @ Q @ z - z.sum())


# ---------------------------------------------------------------------------
# generic box QP  (engine.py:103-133, 248-405)
# ---------------------------------------------------------------------------

def qp_residuals(H, c, A, b, lo, hi, x, y):
    """engine.py:259-281 -> (primal_inf, dual, primal_l1)."""
    if A is not None:
        rr = A @ x - b
        pinf = float(np.max(np.abs(rr))) if rr.size else 0.0
        pl1 = float(np.sum(np.abs(rr)))
    else:
        pinf = pl1 = 0.0
    grad = c.copy()
    if H is not None:
        grad = grad + H @ x
    if A is not None:
        grad = grad - A.T @ y
    dual = float(np.max(np.abs(np.clip(x - grad, lo, hi) - x))) if x.size else 0.0
    return pinf, dual, pl1


def qp_solve(c, H=None, A=None, b=None, lower=None, upper=None, mode: str = RAC,
             block_size: int = 100, beta: float = 1.0, max_iters: int = 100,
             tol_primal: float = 1e-6, tol_dual: float = 1e-6, seed: int = 0,
             fixed_iterations: bool = False,
             on_sweep: Optional[Callable] = None) -> dict:
    """engine.py:322-405 (solve) with run_sweep (284-315).

    `on_sweep(k, blocks, x, y)` observes each sweep (the reference's
    sweep_hook plus the block lists).
    """
    c = np.asarray(c, dtype=float)
    n = c.size
    lo = np.full(n, -np.inf) if lower is None else np.asarray(lower, dtype=float)
    hi = np.full(n, np.inf) if upper is None else np.asarray(upper, dtype=float)
    m = 0 if A is None else A.shape[0]
    rng = np.random.default_rng(seed)
    x = np.clip(np.zeros(n), lo, hi)
    y = np.zeros(m)
    fixed_part = mode in (RP, CYCLIC)
    orders = sweep_orders(mode, rng, n, block_size)
    chol_cache: dict = {}
    p0, _, _ = qp_residuals(H, c, A, b, lo, hi, x, y)
    bar = DIVERGENCE_FACTOR * max(p0, 1.0)
    ph, pl1h, dh = [], [], []
    status = "max_iters"
    sweeps = 0
    converged_early = False
    for _ in range(max_iters):
        blocks = next(orders)
        x = x.copy()
        for idx in blocks:
            Mb = np.zeros((idx.size, idx.size))
            Hb = Hbb = Ab = None
            if H is not None:
                Hb = H[:, idx]
                Hbb = Hb[idx, :]
                Mb = Mb + Hbb
            if A is not None:
                Ab = A[:, idx]
                Mb = Mb + beta * (Ab.T @ Ab)
            xb = x[idx]
            rhs = -c[idx]
            if Hb is not None:
                rhs = rhs - (Hb.T @ x - Hbb @ xb)
            if Ab is not None:
                rest = A @ x - Ab @ xb
                rhs = rhs + Ab.T @ y - beta * (Ab.T @ (rest - b))
            L = None
            if fixed_part:
                key = idx.tobytes()
                L = chol_cache.get(key)
                if L is None:
                    L = _chol(Mb)
                    chol_cache[key] = L
            x[idx] = box_block_min(Mb, rhs, lo[idx], hi[idx], L=L)
        if A is not None:
            y = y - beta * (A @ x - b)
        sweeps += 1
        if on_sweep is not None:
            on_sweep(sweeps, blocks, x, y)
        pinf, dual, pl1 = qp_residuals(H, c, A, b, lo, hi, x, y)
        ph.append(pinf)
        pl1h.append(pl1)
        dh.append(dual)
        if pinf > bar:
            status = "diverged"
            converged_early = True
            break
        if not fixed_iterations and pinf <= tol_primal and dual <= tol_dual:
            status = "converged"
            converged_early = True
            break
    if not converged_early and ph and ph[-1] <= tol_primal and dh[-1] <= tol_dual:
        status = "converged"
    return dict(x=x, y=y, iterations=sweeps, status=status,
                primal_history=np.asarray(ph), primal_l1_history=np.asarray(pl1h),
                dual_history=np.asarray(dh))


def qp_objective(H, c, x) -> float:
    """1/2 x'Hx + c'x."""
    val = float(c @ x)
    if H is not None:
        val += 0.5 * float(x @ (H @ x))
    return val


# ---------------------------------------------------------------------------
# two-block consensus baseline  (elastic_net.py:252-316)
# ---------------------------------------------------------------------------

def consensus_fit(X, y, lam: float, alpha: float, gamma: Optional[float] = None, block_size: int = 100,
                  iters: int = 10, seed: int = 0, tol: Optional[float] = None) -> dict:
    """elastic_net.py:252-316 (consensus_fit): one coefficient copy per sample group
    (direct p x p Cholesky when the group has >= p samples, else the Woodbury n_i x n_i
    route), z shrunk against the aggregated copies, dual ascent per copy."""
    X = np.asarray(X.todense() if hasattr(X, "todense") else X, dtype=float)
    n, p = X.shape
    y = np.asarray(y, dtype=float)
    g = auto_gamma(lam, gamma, X)
    rng = np.random.default_rng(seed)
    want = min(n, max(2, math.ceil(p / min(block_size, p))))
    groups = sorted_chunks(rng.permutation(n), math.ceil(n / want))
    solvers, targets = [], []
    for idx in groups:
        Xi = X[idx]
        targets.append(Xi.T @ y[idx] / n)
        if p <= idx.size:
            solvers.append(("direct", Xi, np.linalg.cholesky(Xi.T @ Xi / n + g * np.eye(p))))
        else:
            solvers.append(("woodbury", Xi, np.linalg.cholesky(Xi @ Xi.T + n * g * np.eye(idx.size))))
    N = len(groups)
    copies, duals, z = np.zeros((N, p)), np.zeros((N, p)), np.zeros(p)
    done, resid = 0, math.inf
    for _ in range(iters):
        for i, ((kind, Xi, L), w0) in enumerate(zip(solvers, targets)):
            w = w0 + duals[i] + g * z
            if kind == "direct":
                copies[i] = scipy.linalg.cho_solve((L, True), w)
            else:
                copies[i] = (w - Xi.T @ scipy.linalg.cho_solve((L, True), Xi @ w)) / g
        agg = duals.sum(axis=0) - g * copies.sum(axis=0)
        z = neg_shrink(agg, lam * alpha) / ((1.0 - alpha) * lam + N * g)
        duals -= g * (copies - z)
        done += 1
        resid = float(np.mean(np.sum(np.abs(copies - z), axis=1)))
        if tol is not None and resid <= tol:
            break
    return dict(beta=copies.mean(axis=0), z=z, xi=duals.mean(axis=0), gamma=g, iterations=done, residual=resid)
