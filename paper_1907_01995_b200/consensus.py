"""Two-block consensus baseline on one B200 — drop-in for racml.elastic_net.consensus_fit.

The paper's Table-1 comparison method (elastic_net.py:252-316): samples are split into
N groups, each keeps a full coefficient copy tied to the shared z.  The once-per-fit
group systems (X_i'X_i/n + gamma I, or the Woodbury form X_i X_i' + n gamma I when a group
has fewer samples than features) are formed and inverted on the device with cuBLAS /
cuSOLVER through torch (a one-time setup, like the reference's np.linalg.cholesky); every
sweep — copy solves, the z shrink, the dual step and the residual — runs in the native
kernels of csrc/consensus.cu (`rac_consensus_run`), batches of 16 sweeps per host poll.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import scipy.sparse as sp
import torch

from . import _device, _native
from .elastic_net import ElasticNetModel, ElasticNetSpec, resolve_gamma
from .problems import Matrix, chunk_indices


class _Args(C.Structure):
    _fields_ = [("N", C.c_int32), ("p", C.c_int64), ("kind", C.c_void_p), ("ni", C.c_void_p),
                ("off_inv", C.c_void_p), ("off_x", C.c_void_p), ("off_u", C.c_void_p), ("inv", C.c_void_p),
                ("xg", C.c_void_p), ("w0", C.c_void_p), ("copies", C.c_void_p), ("duals", C.c_void_p),
                ("z", C.c_void_p), ("u", C.c_void_p), ("inner", C.c_void_p), ("part", C.c_void_p),
                ("hist", C.c_void_p), ("state", C.c_void_p), ("wb_rows", C.c_int64),
                ("direct_groups", C.c_int32), ("part_cap", C.c_int32), ("gamma", C.c_double),
                ("thr", C.c_double), ("denom", C.c_double), ("tol", C.c_double)]


def _spd_inverse(M: torch.Tensor) -> torch.Tensor:
    """Inverse of an SPD matrix through its Cholesky factor (cuSOLVER); a failed factorization
    raises numpy's LinAlgError like the reference's np.linalg.cholesky (elastic_net.py:286,290)."""
    L, info = torch.linalg.cholesky_ex(M)
    if int(info.item()) != 0:
        raise np.linalg.LinAlgError("Matrix is not positive definite")
    return torch.cholesky_inverse(L)


def consensus_fit(X: Matrix, y: np.ndarray, spec: ElasticNetSpec, *, batch: int = 16,
                  device=None) -> ElasticNetModel:
    """Two-block consensus fit (elastic_net.py:252-316): same arguments, groups, stopping and
    returned fields as the reference."""
    spec.validate()
    n, p = X.shape
    y = np.asarray(y, dtype=float)
    gamma = resolve_gamma(spec, X)
    rng = np.random.default_rng(spec.seed)
    copies_wanted = min(n, max(2, math.ceil(p / min(spec.block_size, p))))
    groups = [np.asarray(g, dtype=np.int64) for g in chunk_indices(rng.permutation(n), math.ceil(n / copies_wanted))]
    N = len(groups)
    dev = _device.require_cuda(device)
    lib = _native.load()
    with torch.cuda.device(dev):
        Xd = _device.upload(np.asarray(X.todense(), dtype=float) if sp.issparse(X) else np.asarray(X, dtype=float),
                            device=dev)
        yd = _device.upload(y, device=dev)
        kinds, nis, off_inv, off_x, off_u = [], [], [], [], []
        invs, xgs, w0 = [], [], torch.empty((N, p), dtype=torch.float64, device=dev)
        pos_inv = pos_x = pos_u = 0
        eye_p = None
        for i, idx in enumerate(groups):
            it = torch.from_numpy(idx).to(dev)
            Xi = Xd.index_select(0, it)
            w0[i] = Xi.T @ yd[it] / n
            ni = idx.size
            nis.append(ni)
            off_u.append(pos_u)
            if p <= ni:
                if eye_p is None:
                    eye_p = torch.eye(p, dtype=torch.float64, device=dev)
                inv = _spd_inverse(Xi.T @ Xi / n + gamma * eye_p)
                kinds.append(0)
                off_x.append(0)
            else:
                inv = _spd_inverse(Xi @ Xi.T + n * gamma * torch.eye(ni, dtype=torch.float64, device=dev))
                kinds.append(1)
                off_x.append(pos_x)
                xgs.append(Xi.reshape(-1))
                pos_x += ni * p
                pos_u += ni
            off_inv.append(pos_inv)
            invs.append(inv.reshape(-1))
            pos_inv += inv.numel()
        inv_all = torch.cat(invs)
        xg = torch.cat(xgs) if xgs else torch.zeros(1, dtype=torch.float64, device=dev)
        wb_rows = pos_u
        i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)   # noqa: E731
        i64 = lambda v: torch.tensor(v, dtype=torch.int64, device=dev)   # noqa: E731
        kind_t, ni_t, offi_t, offx_t, offu_t = i32(kinds), i32(nis), i64(off_inv), i64(off_x), i64(off_u)
        copies = torch.zeros((N, p), dtype=torch.float64, device=dev)
        duals = torch.zeros((N, p), dtype=torch.float64, device=dev)
        z = torch.zeros(p, dtype=torch.float64, device=dev)
        u = torch.zeros(max(wb_rows, 1), dtype=torch.float64, device=dev)
        inner = torch.zeros_like(u)
        part_cap = 4096
        part = torch.zeros(part_cap, dtype=torch.float64, device=dev)
        hist = torch.zeros(max(spec.iters, 1), dtype=torch.float64, device=dev)
        state = torch.zeros(2, dtype=torch.int32, device=dev)
        args = _Args(N=N, p=p, kind=kind_t.data_ptr(), ni=ni_t.data_ptr(), off_inv=offi_t.data_ptr(),
                     off_x=offx_t.data_ptr(), off_u=offu_t.data_ptr(), inv=inv_all.data_ptr(), xg=xg.data_ptr(),
                     w0=w0.data_ptr(), copies=copies.data_ptr(), duals=duals.data_ptr(), z=z.data_ptr(),
                     u=u.data_ptr(), inner=inner.data_ptr(), part=part.data_ptr(), hist=hist.data_ptr(),
                     state=state.data_ptr(), wb_rows=wb_rows, direct_groups=int(sum(k == 0 for k in kinds)),
                     part_cap=part_cap, gamma=float(gamma), thr=float(spec.lam * spec.alpha),
                     denom=float((1.0 - spec.alpha) * spec.lam + N * gamma),
                     tol=-1.0 if spec.tol is None else float(spec.tol))
        stream = _device.stream_handle(device=dev)
        done = 0
        while done < spec.iters:
            k = min(batch, spec.iters - done)
            _native.check(lib.rac_consensus_run(C.byref(args), k, stream))
            done += k
            if spec.tol is not None and int(state[1].item()):
                break
        iterations = int(state[0].item())
        residual = float(hist[iterations - 1].item()) if iterations else math.inf
        return ElasticNetModel(beta=copies.mean(dim=0).cpu().numpy(), z=z.cpu().numpy(),
                               xi=duals.mean(dim=0).cpu().numpy(), spec=spec, gamma=gamma,
                               iterations=iterations, residual=residual)
