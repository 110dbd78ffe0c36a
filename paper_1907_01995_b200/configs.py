"""Seeded synthetic inputs for the five BASELINE.json configurations.

BASELINE.json names no public dataset; these generators follow the pinned
recipe of SURVEY.md §8(d) (one ``np.random.default_rng(0)`` per config,
drawn in a fixed order).  Each returns the arrays exactly as they are passed
to the reference-signature entry point, plus the call arguments, so the CPU
oracle and the GPU path see byte-identical inputs.

Scaling decisions:
  * configs 2 and 5 solve the unnormalized LASSO 1/2||y - D b||^2 + lam||b||_1
    and are realized through ``fit`` by pre-scaling (sqrt(m) D, sqrt(m) y);
  * config 3's lambda carries the explicit /m;
  * config 4 runs ``train`` with the linear kernel and beta = 1.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

CONFIG_NAMES = {
    1: "ridge_2000x500_s50",
    2: "lasso_10000x2000_s100",
    3: "elasticnet_50000x5000_s200",
    4: "svm_dual_linear_N20000_d500_s100",
    5: "hd_lasso_5000x100000_s500",
}


@dataclass
class EnCase:
    """Inputs for ``elastic_net.fit`` (X is m x n, C-order float64)."""
    name: str
    X: np.ndarray
    y: np.ndarray
    lam: float
    alpha: float
    gamma: float
    block_size: int
    iters: int
    tol: float | None
    seed: int = 0
    extra: dict = field(default_factory=dict)


@dataclass
class SvmCase:
    """Inputs for ``svm.train`` (X is N x d)."""
    name: str
    X: np.ndarray
    labels: np.ndarray
    C: float
    block_size: int
    beta: float
    max_iters: int
    tol_primal: float
    tol_dual: float
    seed: int = 0


def config1(scale: float = 1.0) -> EnCase:
    rng = np.random.default_rng(0)
    m, n = int(2000 * scale), int(500 * scale)
    D = rng.standard_normal((m, n))
    b = rng.standard_normal(n)
    y = D @ b + 0.1 * rng.standard_normal(m)
    return EnCase(CONFIG_NAMES[1], D, y, lam=1e-3, alpha=0.0, gamma=1.0,
                  block_size=50, iters=200, tol=None)


def config2(scale: float = 1.0) -> EnCase:
    rng = np.random.default_rng(0)
    m, n = int(10000 * scale), int(2000 * scale)
    D = rng.standard_normal((m, n))
    D /= np.linalg.norm(D, axis=0)
    k = max(1, int(round(0.05 * n)))
    support = rng.choice(n, k, replace=False)
    b = np.zeros(n)
    b[support] = rng.standard_normal(k)
    y = D @ b + 0.01 * rng.standard_normal(m)
    lam = 0.1 * float(np.max(np.abs(D.T @ y)))
    sm = math.sqrt(m)
    return EnCase(CONFIG_NAMES[2], sm * D, sm * y, lam=lam, alpha=1.0, gamma=1.0,
                  block_size=100, iters=2000, tol=1e-6)


def config3(scale: float = 1.0) -> EnCase:
    rng = np.random.default_rng(0)
    m, n = int(50000 * scale), int(5000 * scale)
    E = rng.standard_normal((m, n))
    D = np.empty_like(E)
    D[:, 0] = E[:, 0]
    w = math.sqrt(0.75)
    for j in range(1, n):
        D[:, j] = 0.5 * D[:, j - 1] + w * E[:, j]
    del E
    k = max(1, int(round(0.02 * n)))
    support = rng.choice(n, k, replace=False)
    b = np.zeros(n)
    b[support] = rng.choice([-1.0, 1.0], k) * rng.uniform(1.0, 3.0, k)
    y = D @ b + 0.5 * rng.standard_normal(m)
    lam = 0.05 * float(np.max(np.abs(D.T @ y))) / m
    return EnCase(CONFIG_NAMES[3], D, y, lam=lam, alpha=0.5, gamma=1.0,
                  block_size=200, iters=1000, tol=1e-6)


def config4(scale: float = 1.0, max_iters: int = 10000) -> SvmCase:
    rng = np.random.default_rng(0)
    N, d = int(20000 * scale), int(500 * scale) if scale < 1 else 500
    labels = np.where(np.arange(N) < N // 2, 1.0, -1.0)
    X = rng.standard_normal((N, d)) + labels[:, None] * (0.3 / math.sqrt(d))
    flip = rng.choice(N, max(1, int(round(0.05 * N))), replace=False)
    labels[flip] *= -1.0
    return SvmCase(CONFIG_NAMES[4], X, labels, C=1.0, block_size=100, beta=1.0,
                   max_iters=max_iters, tol_primal=1e-6, tol_dual=1e-6)


def config5(scale: float = 1.0) -> EnCase:
    rng = np.random.default_rng(0)
    m, n = int(5000 * scale), int(100000 * scale)
    D = rng.standard_normal((m, n)) / math.sqrt(m)
    k = max(1, int(round(0.01 * n)))
    support = rng.choice(n, k, replace=False)
    b = np.zeros(n)
    b[support] = rng.standard_normal(k)
    y = D @ b + 0.01 * rng.standard_normal(m)
    lam = 0.05 * float(np.max(np.abs(D.T @ y)))
    sm = math.sqrt(m)
    return EnCase(CONFIG_NAMES[5], sm * D, sm * y, lam=lam, alpha=1.0, gamma=1.0,
                  block_size=500, iters=1000, tol=1e-6)


GENERATORS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
