"""Data model of the RAC sweep — the reference's contract types, re-declared.

Mirrors the names, fields, defaults and validation messages of
racml.problems (problems.py:90-375) so callers of the reference can switch
imports.  Block assembly on the hot path runs on the device
(`rac_chunk_sort`); `chunk_indices` here is the host-side API twin.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import Optional, Union

import numpy as np
import scipy.sparse as sp

Matrix = Union[np.ndarray, sp.spmatrix]


class Mode(str, Enum):
    """Block assembly policy (problems.py:318-323)."""

    RAC = "rac"        # fresh random partition every sweep
    RP = "rp"          # fixed partition, re-permuted block order every sweep
    CYCLIC = "cyclic"  # fixed partition, fixed order


class Status(str, Enum):
    """Termination status (problems.py:326-329)."""

    CONVERGED = "converged"
    MAX_ITERS = "max_iters"
    DIVERGED = "diverged"


def as_dense(mat: Matrix) -> np.ndarray:
    if sp.issparse(mat):
        return np.asarray(mat.todense(), dtype=float)
    return np.asarray(mat, dtype=float)


def chunk_indices(indices: np.ndarray, block_size: int) -> tuple[tuple[int, ...], ...]:
    """Consecutive chunks of `block_size`, each sorted (problems.py:234-243)."""
    idx = np.asarray(indices)
    out = []
    for lo in range(0, idx.size, block_size):
        out.append(tuple(int(v) for v in np.sort(idx[lo:lo + block_size])))
    return tuple(out)


def _vector(v, name: str) -> np.ndarray:
    arr = np.asarray(v, dtype=float)
    if arr.ndim != 1:
        raise ValueError(f"{name} must be a 1-D vector, got shape {arr.shape}")
    return arr


@dataclass(frozen=True)
class QpProblem:
    """min 1/2 x'Hx + c'x  s.t.  Ax = b, lower <= x <= upper (problems.py:90-132)."""

    c: np.ndarray
    H: Optional[Matrix] = None
    A: Optional[Matrix] = None
    b: Optional[np.ndarray] = None
    lower: Optional[np.ndarray] = None
    upper: Optional[np.ndarray] = None

    def __post_init__(self):
        c = _vector(self.c, "c")
        object.__setattr__(self, "c", c)
        n = c.size
        if self.b is not None:
            object.__setattr__(self, "b", _vector(self.b, "b"))
        object.__setattr__(self, "lower", _vector(self.lower, "lower") if self.lower is not None
                           else np.full(n, -np.inf))
        object.__setattr__(self, "upper", _vector(self.upper, "upper") if self.upper is not None
                           else np.full(n, np.inf))

    @property
    def n(self) -> int:
        return self.c.size

    @property
    def m(self) -> int:
        return 0 if self.A is None else self.A.shape[0]

    @property
    def is_bounded(self) -> bool:
        return bool(np.any(np.isfinite(self.lower)) or np.any(np.isfinite(self.upper)))


@dataclass(frozen=True)
class ValidationReport:
    """Invariant violations found by validate_problem; empty means valid."""

    issues: tuple[str, ...] = ()

    @property
    def ok(self) -> bool:
        return not self.issues

    def __bool__(self) -> bool:
        return self.ok


def _matrix_issues(mat: Matrix, name: str) -> list[str]:
    if sp.issparse(mat):
        csc = mat.tocsc()
        out = []
        if not np.all(np.isfinite(csc.data)):
            out.append(f"{name}: contains non-finite entries")
        return out
    arr = np.asarray(mat)
    if arr.ndim != 2:
        return [f"{name}: expected a 2-D array, got ndim={arr.ndim}"]
    if not np.all(np.isfinite(arr)):
        return [f"{name}: contains non-finite entries"]
    return []


def validate_problem(problem: QpProblem) -> ValidationReport:
    """Collect every QpProblem invariant violation (problems.py:149-188)."""
    issues: list[str] = []
    n = problem.n
    if problem.H is not None:
        issues += _matrix_issues(problem.H, "H")
        if problem.H.shape != (n, n):
            issues.append(f"H: expected shape ({n}, {n}), got {problem.H.shape}")
        elif not issues:
            Hd = as_dense(problem.H)
            scale = max(1.0, float(np.max(np.abs(Hd))) if Hd.size else 1.0)
            if np.max(np.abs(Hd - Hd.T)) > 1e-12 * scale:
                issues.append("H: not symmetric within 1e-12 relative tolerance")
    if problem.A is not None:
        issues += _matrix_issues(problem.A, "A")
        if problem.A.shape[1] != n:
            issues.append(f"A: expected {n} columns, got {problem.A.shape[1]}")
        if problem.b is None:
            issues.append("b: required when A is present")
        elif problem.b.size != problem.A.shape[0]:
            issues.append(f"b: length {problem.b.size} does not match {problem.A.shape[0]} rows of A")
        if problem.b is not None and not np.all(np.isfinite(problem.b)):
            issues.append("b: contains non-finite entries")
    elif problem.b is not None and problem.b.size:
        issues.append("b: present without A")
    if not np.all(np.isfinite(problem.c)):
        issues.append("c: contains non-finite entries")
    for name, v in (("lower", problem.lower), ("upper", problem.upper)):
        if v.size != n:
            issues.append(f"{name}: length {v.size} does not match n={n}")
        if np.any(np.isnan(v)):
            issues.append(f"{name}: contains NaN")
    if problem.lower.size == n and problem.upper.size == n and np.any(problem.lower > problem.upper):
        issues.append("bounds: lower > upper for at least one variable")
    return ValidationReport(tuple(issues))


@dataclass(frozen=True)
class SolverConfig:
    """Sweep solver settings (problems.py:332-354)."""

    mode: Mode = Mode.RAC
    block_size: int = 100
    beta_penalty: float = 1.0
    max_iters: int = 100
    tol_primal: float = 1e-6
    tol_dual: float = 1e-6
    seed: int = 0
    fixed_iterations: bool = False

    def validate(self, n: int) -> None:
        if self.beta_penalty <= 0:
            raise ValueError(f"beta_penalty must be > 0, got {self.beta_penalty}")
        if not (1 <= self.block_size <= n):
            raise ValueError(f"block_size must be in [1, n]; got {self.block_size} with n={n}")
        if self.tol_primal <= 0 or self.tol_dual <= 0:
            raise ValueError("tolerances must be > 0")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")


@dataclass
class SolveResult:
    """Solution, duals, per-sweep residual histories and status (problems.py:357-375)."""

    x: np.ndarray
    y: np.ndarray
    iterations: int
    primal_residual_history: np.ndarray
    primal_l1_history: np.ndarray
    dual_residual_history: np.ndarray
    status: Status

    @property
    def primal_residual(self) -> float:
        return float(self.primal_residual_history[-1]) if self.iterations else math.inf

    @property
    def dual_residual(self) -> float:
        return float(self.dual_residual_history[-1]) if self.iterations else math.inf
