"""Generic box-QP RAC sweep on one B200 — drop-in for racml.engine.solve.

    min 1/2 x'Hx + c'x   s.t.  Ax = b,  lower <= x <= upper

Same signature, validation, modes (RAC / RP / CYCLIC), sweep_hook,
SolveResult fields, divergence guard and for-else convergence rule as
engine.py:322-405.  Block systems, the Gauss-Seidel chain, the exact box
block solver, the dual step and the residuals all run in the native engine
(`rac_qp_*`, include/rac_b200.h).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.sparse as sp
import torch

from . import _device, _native
from .problems import Mode, QpProblem, SolveResult, SolverConfig, Status, as_dense, validate_problem

DIVERGENCE_FACTOR = 1e8       # engine.py:34
ACTIVE_SET_PASS_FACTOR = 10   # engine.py:38
PG_TOL = 1e-10                # engine.py:39

_MODE = {Mode.RAC: _native.MODE_RAC, Mode.RP: _native.MODE_RP, Mode.CYCLIC: _native.MODE_CYCLIC}
_STATUS = {_native.STATUS_MAX_ITERS: Status.MAX_ITERS, _native.STATUS_CONVERGED: Status.CONVERGED,
           _native.STATUS_DIVERGED: Status.DIVERGED}


class BlockDefinitenessError(ArithmeticError):
    """A block subsystem H_bb + beta A_b'A_b was not positive definite (engine.py:42-48)."""


NOT_PD_MESSAGE = ("block matrix H_bb + beta*A_b'A_b is not positive definite; "
                  "the solver's block positive-definiteness assumption is violated")


class QpSolver:
    """One native dense box-QP sweep context (rac_qp_ctx) on the current stream."""

    def __init__(self, n: int, m: int, block_size: int, mode: Mode, beta: float,
                 ridge_rel: float = 0.0, device=None):
        self.dev = _device.require_cuda(device)
        self.lib = _native.load()
        self.n, self.m, self.s = int(n), int(m), int(block_size)
        self.p = -(-self.n // self.s)
        self.mode = Mode(mode)
        h = _native._p()
        with torch.cuda.device(self.dev):    # the context allocates and launches on this device
            _native.check(self.lib.rac_qp_create(h, self.n, self.m, self.s, _MODE[self.mode], float(beta),
                                                 float(ridge_rel), _device.stream_handle(device=self.dev)))
        self.h = h
        self._keep = []

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.rac_qp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_problem(self, c, lower, upper, H=None, A=None, b=None, borrowed_h: torch.Tensor | None = None):
        up = lambda v: None if v is None else _device.upload(v, device=self.dev)  # noqa: E731
        cd, lo, hi, Hd, Ad, bd = up(c), up(lower), up(upper), up(H), up(A), up(b)
        if borrowed_h is not None:
            _native.check(self.lib.rac_qp_borrow_h(self.h, borrowed_h.data_ptr()))
        _native.check(self.lib.rac_qp_set_problem(
            self.h, _device.ptr(Hd), _device.ptr(Ad), _device.ptr(bd), cd.data_ptr(), lo.data_ptr(),
            hi.data_ptr()))
        self._keep = [cd, lo, hi, Hd, Ad, bd, borrowed_h]

    def set_kernel_strips(self, X: np.ndarray, labels: np.ndarray, kind: int, sigma: float, max_strip_bytes: int):
        """No resident n x n H: per sweep the blocks' H_bb and batches of strip rows are formed
        from the samples (rac_qp_set_kernel_strips; before set_problem)."""
        Xd = _device.upload(np.ascontiguousarray(X, dtype=float), device=self.dev)
        yd = _device.upload(np.asarray(labels, dtype=float), device=self.dev)
        _native.check(self.lib.rac_qp_set_kernel_strips(self.h, Xd.data_ptr(), int(X.shape[1]), yd.data_ptr(),
                                                        int(kind), float(sigma), int(max_strip_bytes)))
        self._strip_keep = [Xd, yd]

    def set_divergence_bar(self, bar: float):
        _native.check(self.lib.rac_qp_set_divergence_bar(self.h, float(bar)))

    def set_partition(self, perm: np.ndarray):
        pd = _device.upload(np.asarray(perm, dtype=np.int64), dtype=torch.int64, device=self.dev)
        _native.check(self.lib.rac_qp_set_partition(self.h, pd.data_ptr()))
        self._keep.append(pd)

    def run(self, perms_dev: Optional[torch.Tensor], count: int, tol_p: float, tol_d: float, fixed: bool):
        _native.check(self.lib.rac_qp_run(self.h, _device.ptr(perms_dev), int(count), float(tol_p),
                                          float(tol_d), int(bool(fixed))))

    def progress(self):
        it, st, fb = _native._i32(), _native._i32(), _native._i32()
        _native.check(self.lib.rac_qp_progress(self.h, it, st, fb))
        return it.value, _STATUS[st.value], fb.value

    def state(self):
        x = torch.empty(self.n, dtype=torch.float64, device=self.dev)
        y = torch.empty(max(self.m, 1), dtype=torch.float64, device=self.dev)
        hx = torch.empty_like(x)
        _native.check(self.lib.rac_qp_get(self.h, x.data_ptr(), y.data_ptr(), hx.data_ptr(), None))
        return x, y[:self.m], hx

    def history(self, count: int):
        bufs = [torch.empty(max(count, 1), dtype=torch.float64, device=self.dev) for _ in range(3)]
        _native.check(self.lib.rac_qp_history(self.h, *(b.data_ptr() for b in bufs), count))
        return [b[:count] for b in bufs]


def drive(solver: QpSolver, rng: np.random.Generator, max_iters: int, tol_p: float, tol_d: float,
          fixed: bool, hook=None, batch: int = 16):
    """Run sweeps with the reference's RNG call order until done; returns (iterations, status)."""
    n, p = solver.n, solver.p
    if solver.mode == Mode.RAC:
        feeder = _device.PermutationFeeder(rng, n, solver.dev)
    elif solver.mode == Mode.RP:
        feeder = _device.PermutationFeeder(rng, p, solver.dev)
    else:
        feeder = None
    step = 1 if hook is not None else max(1, batch)
    done = 0
    it, status, failed = 0, Status.MAX_ITERS, -1
    def draw(count):
        return feeder.draw(count) if feeder is not None and count > 0 else None

    perms = draw(min(step, max_iters))
    while done < max_iters:
        k = min(step, max_iters - done)
        solver.run(perms, k, tol_p, tol_d, fixed)
        done += k
        # the next batch's permutations are drawn while the device runs this one (same
        # PCG64 order; a batch drawn past the stop is dropped)
        perms = draw(min(step, max_iters - done))
        it, status, failed = solver.progress()
        if failed >= 0:
            raise BlockDefinitenessError(NOT_PD_MESSAGE)
        if hook is not None and it == done:
            x, y, _ = solver.state()
            hook(it, x.cpu().numpy(), y.cpu().numpy())
        if status != Status.MAX_ITERS:
            break
    return it, status


def solve(problem: QpProblem, config: SolverConfig, sweep_hook=None, *, device=None) -> SolveResult:
    """Run the randomized multi-block sweep until tolerance or iteration cap (engine.py:322-405).

    `device` (not in the reference): CUDA device index, default the current device."""
    report = validate_problem(problem)
    if not report.ok:
        raise ValueError("invalid problem: " + "; ".join(report.issues))
    n = problem.n
    config.validate(n)
    dev = _device.require_cuda(device)
    with torch.cuda.device(dev):
        return _solve_on(dev, problem, config, sweep_hook)


def _solve_on(dev, problem: QpProblem, config: SolverConfig, sweep_hook) -> SolveResult:
    n = problem.n
    mode = Mode(config.mode)
    rng = np.random.default_rng(config.seed)
    H = None if problem.H is None else as_dense(problem.H)
    A = None if problem.A is None else as_dense(problem.A)
    m = 0 if A is None else A.shape[0]
    solver = QpSolver(n, m, config.block_size, mode, config.beta_penalty, 0.0, device=dev)
    try:
        solver.set_problem(problem.c, problem.lower, problem.upper, H=H, A=A,
                           b=None if m == 0 else problem.b)
        if mode == Mode.CYCLIC:
            solver.set_partition(np.arange(n))
        elif mode == Mode.RP:
            solver.set_partition(rng.permutation(n))
        it, status = drive(solver, rng, config.max_iters, config.tol_primal, config.tol_dual,
                           config.fixed_iterations, hook=sweep_hook)
        x, y, _ = solver.state()
        hp, hl, hd = (h.cpu().numpy() for h in solver.history(it))
        if status == Status.MAX_ITERS and it and hp[-1] <= config.tol_primal and hd[-1] <= config.tol_dual:
            status = Status.CONVERGED   # engine.py:392-397 (for-else)
        return SolveResult(x=x.cpu().numpy(), y=y.cpu().numpy(), iterations=it,
                           primal_residual_history=hp, primal_l1_history=hl,
                           dual_residual_history=hd, status=status)
    finally:
        solver.close()


@dataclass
class BlockSystem:
    """One block's subproblem min 1/2 x'Mx - r'x over a box (engine.py:51-65).  `bounded`
    defaults to "some bound is finite", as in the reference."""

    matrix: np.ndarray
    rhs: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    bounded: Optional[bool] = None

    def __post_init__(self):
        if self.bounded is None:
            self.bounded = bool(np.any(np.isfinite(self.lower)) or np.any(np.isfinite(self.upper)))


@dataclass(frozen=True)
class ResidualPair:
    """Primal ||Ax - b||_inf, box-projected stationarity (inf-norms) and ||Ax - b||_1
    (engine.py:68-77)."""

    primal: float
    dual: float
    primal_l1: float


def _box_min_device(M: torch.Tensor, r: torch.Tensor, lo: torch.Tensor, hi: torch.Tensor) -> torch.Tensor:
    lib = _native.load()
    s = int(r.numel())
    x = torch.empty(s, dtype=torch.float64, device=M.device)
    info = torch.zeros(1, dtype=torch.int32, device=M.device)
    _native.check(lib.rac_box_block_min(M.data_ptr(), r.data_ptr(), lo.data_ptr(), hi.data_ptr(), s,
                                        x.data_ptr(), info.data_ptr(), _device.stream_handle(device=M.device)))
    if int(info.item()) != 0:
        raise BlockDefinitenessError(NOT_PD_MESSAGE)
    return x


def solve_block(system, chol: Optional[np.ndarray] = None, *legacy, device=None) -> np.ndarray:
    """Exact minimizer of 1/2 x'Mx - r'x over the block's box, on the device
    (engine.py:189-245: Cholesky solve; bounded blocks run the clamp / release-worst
    active set with the 10 s pass budget and the projected-gradient fallback — csrc/boxqp.cuh).

    `chol` (the reference's cached factor) is accepted for signature compatibility; the
    device factors M itself (same factor up to rounding).  An unbounded system
    (`bounded=False`) is the plain SPD solve.  The array form
    solve_block(M, r, lower, upper) is kept for the native tests."""
    if not isinstance(system, BlockSystem):
        if chol is None or len(legacy) != 2:
            raise TypeError("solve_block(system: BlockSystem, chol=None)")
        system = BlockSystem(np.asarray(system, dtype=float), np.asarray(chol, dtype=float),
                             np.asarray(legacy[0], dtype=float), np.asarray(legacy[1], dtype=float))
    dev = _device.require_cuda(device)
    s = int(np.asarray(system.rhs).size)
    lo, hi = np.asarray(system.lower, dtype=float), np.asarray(system.upper, dtype=float)
    if not system.bounded:
        lo, hi = np.full(s, -np.inf), np.full(s, np.inf)
    with torch.cuda.device(dev):
        M = _device.upload(np.asarray(system.matrix, dtype=float), device=dev)
        r, lod, hid = (_device.upload(v, device=dev) for v in (np.asarray(system.rhs, dtype=float), lo, hi))
        return _box_min_device(M, r, lod, hid).cpu().numpy()


def _dense_dev(mat, dev):
    return None if mat is None else _device.upload(as_dense(mat), device=dev)


def dual_update(y: np.ndarray, A, x: np.ndarray, b: np.ndarray, beta: float, *, device=None) -> np.ndarray:
    """y - beta (Ax - b) (engine.py:248-256), on the device."""
    if A is None:
        return np.asarray(y, dtype=float).copy()
    dev = _device.require_cuda(device)
    with torch.cuda.device(dev):
        Ad = _dense_dev(A, dev)
        r = Ad @ _device.upload(np.asarray(x, dtype=float), device=dev) - _device.upload(np.asarray(b, dtype=float),
                                                                                        device=dev)
        yv = np.asarray(y, dtype=float)
        if yv.size != r.numel():
            raise ValueError(f"y has length {yv.size}, expected {r.numel()}")
        return (_device.upload(yv, device=dev) - beta * r).cpu().numpy()


def compute_residuals(problem: QpProblem, x: np.ndarray, y: np.ndarray, *, device=None) -> ResidualPair:
    """Primal ||Ax - b||_inf (and 1-norm) and the box-projected stationarity step
    ||P(x - (Hx + c - A'y)) - x||_inf (engine.py:259-281), on the device.  NaN propagates
    (as numpy's max does)."""
    dev = _device.require_cuda(device)
    with torch.cuda.device(dev):
        xd = _device.upload(np.asarray(x, dtype=float), device=dev)
        grad = _device.upload(problem.c, device=dev).clone()
        primal = primal_l1 = 0.0
        if problem.A is not None:
            Ad = _dense_dev(problem.A, dev)
            r = Ad @ xd - _device.upload(problem.b, device=dev)
            if r.numel():
                primal = float(r.abs().max().item())
                primal_l1 = float(r.abs().sum().item())
            grad -= Ad.T @ _device.upload(np.asarray(y, dtype=float), device=dev)
        if problem.H is not None:
            grad += _dense_dev(problem.H, dev) @ xd
        v = xd - grad
        proj = torch.minimum(torch.maximum(v, _device.upload(problem.lower, device=dev)),
                             _device.upload(problem.upper, device=dev))
        proj = torch.where(torch.isnan(v), v, proj)
        dual = float((proj - xd).abs().max().item()) if xd.numel() else 0.0
        return ResidualPair(primal=primal, dual=dual, primal_l1=primal_l1)


def assemble_block_system(problem: QpProblem, x: np.ndarray, y: np.ndarray, block, beta: float, *,
                          device=None) -> BlockSystem:
    """The exact subproblem of one block with the others fixed (engine.py:136-157):
    M = H_bb + beta A_b'A_b,  r = -(c_b + H_{b,rest} x_rest - A_b'y + beta A_b'(A_rest x_rest - b)),
    gathered on the device (no permuted copy of H or A)."""
    n = problem.n
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    if x.size != n:
        raise ValueError(f"x has length {x.size}, expected {n}")
    if y.size != problem.m:
        raise ValueError(f"y has length {y.size}, expected {problem.m}")
    idx_np = np.asarray(block, dtype=np.int64)
    dev = _device.require_cuda(device)
    with torch.cuda.device(dev):
        idx = torch.from_numpy(idx_np).to(dev)
        xd = _device.upload(x, device=dev)
        xb = xd[idx]
        s = idx.numel()
        M = torch.zeros((s, s), dtype=torch.float64, device=dev)
        rhs = -_device.upload(problem.c, device=dev)[idx]
        if problem.H is not None:
            Hb = _dense_dev(problem.H, dev)[:, idx]         # columns of symmetric H
            Hbb = Hb[idx, :]
            M += Hbb
            rhs -= Hb.T @ xd - Hbb @ xb
        if problem.A is not None:
            Ad = _dense_dev(problem.A, dev)
            Ab = Ad[:, idx]
            M += beta * (Ab.T @ Ab)
            ax_rest = Ad @ xd - Ab @ xb
            rhs += Ab.T @ _device.upload(y, device=dev) - beta * (Ab.T @ (ax_rest - _device.upload(problem.b,
                                                                                                    device=dev)))
        lower, upper = problem.lower[idx_np], problem.upper[idx_np]
        return BlockSystem(matrix=M.cpu().numpy(), rhs=rhs.cpu().numpy(), lower=lower, upper=upper)


def run_sweep(problem: QpProblem, x: np.ndarray, y: np.ndarray, order, beta: float,
              chol_cache: Optional[dict] = None, piece_cache: Optional[dict] = None, *,
              device=None) -> tuple[np.ndarray, np.ndarray]:
    """One full pass in the given block order, then one dual step (engine.py:284-315),
    through the native sweep (rac_qp_set_state + one fixed-partition sweep).

    The blocks must be what chunk_indices produces (equal sizes except a shorter last
    block; indices within a block in any order — the device sorts them, which only
    reorders a block's coordinates).  `chol_cache` / `piece_cache` are accepted for
    signature compatibility; the device forms the block factors itself.  Inputs are not
    modified."""
    groups = [np.asarray(g, dtype=np.int64) for g in order]
    n = problem.n
    if not groups or sum(g.size for g in groups) != n or \
            not np.array_equal(np.sort(np.concatenate(groups)), np.arange(n)):
        raise ValueError("order must partition range(n)")
    s = groups[0].size
    if any(g.size != s for g in groups[:-1]) or groups[-1].size > s:
        raise ValueError("run_sweep on the device needs chunk_indices-shaped blocks (equal sizes, last shorter)")
    report = validate_problem(problem)
    if not report.ok:
        raise ValueError("invalid problem: " + "; ".join(report.issues))
    dev = _device.require_cuda(device)
    with torch.cuda.device(dev):
        H = None if problem.H is None else as_dense(problem.H)
        A = None if problem.A is None else as_dense(problem.A)
        m = 0 if A is None else A.shape[0]
        solver = QpSolver(n, m, s, Mode.CYCLIC, beta, 0.0, device=dev)
        try:
            solver.set_problem(problem.c, problem.lower, problem.upper, H=H, A=A, b=None if m == 0 else problem.b)
            solver.set_divergence_bar(math.inf)
            solver.set_partition(np.concatenate(groups))
            xd = _device.upload(np.asarray(x, dtype=float), device=dev)
            yd = _device.upload(np.asarray(y, dtype=float).reshape(-1), device=dev) if m else None
            _native.check(solver.lib.rac_qp_set_state(solver.h, xd.data_ptr(), _device.ptr(yd)))
            solver.run(None, 1, 0.0, 0.0, True)
            it, _, failed = solver.progress()
            if failed >= 0:
                raise BlockDefinitenessError(NOT_PD_MESSAGE)
            xo, yo, _ = solver.state()
            return xo.cpu().numpy(), yo.cpu().numpy()
        finally:
            solver.close()
