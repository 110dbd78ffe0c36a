"""Generic box-QP RAC sweep on one B200 — drop-in for racml.engine.solve.

    min 1/2 x'Hx + c'x   s.t.  Ax = b,  lower <= x <= upper

Same signature, validation, modes (RAC / RP / CYCLIC), sweep_hook,
SolveResult fields, divergence guard and for-else convergence rule as
engine.py:322-405.  Block systems, the Gauss-Seidel chain, the exact box
block solver, the dual step and the residuals all run in the native engine
(`rac_qp_*`, include/rac_b200.h).
"""

from __future__ import annotations

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
                 ridge_rel: float = 0.0, device: int = 0):
        self.dev = _device.require_cuda(device)
        self.lib = _native.load()
        self.n, self.m, self.s = int(n), int(m), int(block_size)
        self.p = -(-self.n // self.s)
        self.mode = Mode(mode)
        h = _native._p()
        _native.check(self.lib.rac_qp_create(h, self.n, self.m, self.s, _MODE[self.mode], float(beta),
                                             float(ridge_rel), _device.stream_handle()))
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


def solve(problem: QpProblem, config: SolverConfig, sweep_hook=None) -> SolveResult:
    """Run the randomized multi-block sweep until tolerance or iteration cap (engine.py:322-405)."""
    report = validate_problem(problem)
    if not report.ok:
        raise ValueError("invalid problem: " + "; ".join(report.issues))
    n = problem.n
    config.validate(n)
    mode = Mode(config.mode)
    rng = np.random.default_rng(config.seed)
    H = None if problem.H is None else as_dense(problem.H)
    A = None if problem.A is None else as_dense(problem.A)
    m = 0 if A is None else A.shape[0]
    solver = QpSolver(n, m, config.block_size, mode, config.beta_penalty, 0.0)
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


def solve_block(matrix: np.ndarray, rhs: np.ndarray, lower: np.ndarray, upper: np.ndarray) -> np.ndarray:
    """Exact box minimizer of 1/2 x'Mx - r'x for one block on the device (engine.py:189-245)."""
    dev = _device.require_cuda(0)
    lib = _native.load()
    s = int(np.asarray(rhs).size)
    M = _device.upload(np.asarray(matrix, dtype=float), device=dev)
    r, lo, hi = (_device.upload(np.asarray(v, dtype=float), device=dev) for v in (rhs, lower, upper))
    x = torch.empty(s, dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(lib.rac_box_block_min(M.data_ptr(), r.data_ptr(), lo.data_ptr(), hi.data_ptr(), s,
                                        x.data_ptr(), info.data_ptr(), _device.stream_handle()))
    if int(info.item()) != 0:
        raise BlockDefinitenessError(NOT_PD_MESSAGE)
    return x.cpu().numpy()
