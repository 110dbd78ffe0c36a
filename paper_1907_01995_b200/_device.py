"""PyTorch plumbing: device buffers, streams and host->device staging.

PyTorch is used only for memory management and streams; all arithmetic of
the sweep runs in the native sm_100a kernels (_native.py).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native


def require_cuda(device: int = 0) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1907_01995_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _native.require_device(device)
    return torch.device("cuda", device)


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


def upload(arr, dtype=torch.float64, device=None, pinned: bool = True) -> torch.Tensor:
    """numpy (or torch) -> contiguous device tensor, staged through pinned memory."""
    if isinstance(arr, torch.Tensor):
        t = arr.to(dtype)
        if t.is_cuda:
            return t.contiguous()
        src = t.contiguous()
    else:
        np_dtype = np.float64 if dtype == torch.float64 else np.int64
        src = torch.from_numpy(np.ascontiguousarray(arr, dtype=np_dtype))
    if pinned and src.numel() * src.element_size() <= (64 << 20):
        return src.pin_memory().to(device or "cuda", non_blocking=True)
    # large one-shot uploads: pinning would cost more than it saves
    return src.to(device or "cuda")


class PermutationFeeder:
    """Draws the reference's per-sweep permutations from the host PCG64 stream.

    RAC draws rng.permutation(n) per sweep (elastic_net.py:195, svm.py:231,
    engine.py:371); RP draws rng.permutation(p) per sweep after one
    rng.permutation(n) for the fixed partition (elastic_net.py:188-198).
    Batches are staged through pinned memory and copied asynchronously on
    the solver stream, so host generation of the next batch overlaps the
    device sweeps of the current one.
    """

    def __init__(self, rng: np.random.Generator, size: int, device):
        self.rng = rng
        self.size = size
        self.device = device

    def draw(self, count: int) -> torch.Tensor:
        host = torch.empty((count, self.size), dtype=torch.int64).pin_memory()
        view = host.numpy()
        for k in range(count):
            view[k] = self.rng.permutation(self.size)
        return host.to(self.device, non_blocking=True)
