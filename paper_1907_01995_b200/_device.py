"""PyTorch plumbing: device buffers, streams and host->device staging.

PyTorch is used only for memory management and streams; all arithmetic of
the sweep runs in the native sm_100a kernels (_native.py).
"""

from __future__ import annotations

import os
import threading

import numpy as np
import torch

from . import _native


def resolve_device(device=None) -> int:
    """Device index: an int, a torch.device, or None = the current CUDA device (so a rank
    that called torch.cuda.set_device(local) gets its own GPU by default)."""
    if isinstance(device, torch.device):
        device = device.index
    if device is None:
        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    return int(device)


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1907_01995_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    idx = resolve_device(device)
    _native.require_device(idx)
    return torch.device("cuda", idx)


def stream_handle(stream: torch.cuda.Stream | None = None, device=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


class _Stager:
    """Ring of pinned staging buffers for large host->device uploads.

    A pageable cudaMemcpy runs at ~11 GB/s on the B200 hosts; copying
    16 MiB chunks into pinned buffers while the previous chunks' DMA is in
    flight runs the host copy and PCIe transfer concurrently (~4x faster for
    the 160 MB - 4 GB design matrices of BASELINE configs 2-5).
    """

    CHUNK = 16 << 20
    SLOTS = 4

    def __init__(self):
        self.bufs = [torch.empty(self.CHUNK, dtype=torch.uint8).pin_memory() for _ in range(self.SLOTS)]
        self.events = [None] * self.SLOTS
        self.lock = threading.Lock()   # one upload at a time owns the ring (concurrent fits)

    def copy(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        with self.lock:
            self._copy(src, dst)

    def _copy(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        sb = src.reshape(-1).view(torch.uint8)
        db = dst.reshape(-1).view(torch.uint8)
        stream = torch.cuda.current_stream(dst.device)
        total = sb.numel()
        for i, off in enumerate(range(0, total, self.CHUNK)):
            k = i % self.SLOTS
            ln = min(self.CHUNK, total - off)
            if self.events[k] is not None:
                self.events[k].synchronize()
            self.bufs[k][:ln].copy_(sb[off:off + ln])
            db[off:off + ln].copy_(self.bufs[k][:ln], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            self.events[k] = ev


_stagers: dict = {}
_STAGE_LOCK = threading.Lock()   # creation of the per-device rings
# uploads above this go through the persistent pinned ring: pinning a fresh multi-MB buffer per
# call (tensor.pin_memory) costs milliseconds whenever torch's host cache has no block of that
# size (measured: 8.8 ms spikes on an 8 MB design after larger fits)
SMALL_UPLOAD = 1 << 20

ROW_CHUNK_BYTES = 16 << 20


class _RowStreamer:
    """A ring of `nbuf` pinned host buffers and device buffers (4 by default,
    RAC_STAGE_BUFS), one copy stream: later row chunks are copied (host memcpy
    into pinned memory, then DMA) while the consumer's kernels for chunk k run on
    the current stream.  Four buffers keep the DMA engine busy: 54 GB/s against
    48 GB/s with two (scripts/micro/ingest_probe.py)."""

    def __init__(self, device, nbuf: int = 2):
        self.device = device
        self.copy_stream = torch.cuda.Stream(device=device)
        self.nbuf = nbuf
        self.host = [None] * nbuf
        self.dev = [None] * nbuf
        self.copied = [None] * nbuf
        self.consumed = [None] * nbuf
        self.lock = threading.Lock()   # one streamed ingest at a time owns the ring

    def run(self, X: np.ndarray, align: int, consume) -> None:
        # the ring's device buffers are reused by the next ingest only after the device-side
        # wait on `consumed` (events are valid across streams and threads)
        with self.lock:
            self._run(X, align, consume)

    def _run(self, X: np.ndarray, align: int, consume) -> None:
        m, n = X.shape
        rows_per = max(align, (ROW_CHUNK_BYTES // (8 * n)) // align * align)
        need = rows_per * n
        for k in range(self.nbuf):
            if self.host[k] is None or self.host[k].numel() < need:
                self.host[k] = torch.empty(need, dtype=torch.float64).pin_memory()
                self.dev[k] = torch.empty(need, dtype=torch.float64, device=self.device)
        main = torch.cuda.current_stream(self.device)
        src = torch.from_numpy(X)
        for i, r0 in enumerate(range(0, m, rows_per)):
            k = i % self.nbuf
            rows = min(rows_per, m - r0)
            if self.copied[k] is not None:
                self.copied[k].synchronize()            # pinned buffer k is free again
            self.host[k][:rows * n].view(rows, n).copy_(src[r0:r0 + rows])
            with torch.cuda.stream(self.copy_stream):
                if self.consumed[k] is not None:
                    self.copy_stream.wait_event(self.consumed[k])   # device buffer k consumed
                self.dev[k][:rows * n].copy_(self.host[k][:rows * n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
                self.copied[k] = ev
            main.wait_event(ev)
            consume(r0, rows, self.dev[k][:rows * n])
            done = torch.cuda.Event()
            done.record(main)
            self.consumed[k] = done


_streamers: dict = {}


def stream_rows(X: np.ndarray, align: int, consume, device=None) -> None:
    """Feed a C-contiguous host matrix to `consume(row0, rows, device_chunk)` in
    row chunks of ~ROW_CHUNK_BYTES (rows a multiple of `align` except the last)."""
    dev = torch.device(device or "cuda")
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    with _STAGE_LOCK:
        if key not in _streamers:
            _streamers[key] = _RowStreamer(torch.device("cuda", key), int(os.environ.get("RAC_STAGE_BUFS", "4")))
        st = _streamers[key]
    st.run(np.ascontiguousarray(X, dtype=np.float64), align, consume)


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
    dev = torch.device(device or "cuda")
    nbytes = src.numel() * src.element_size()
    if not pinned:
        return src.to(dev)
    if nbytes <= SMALL_UPLOAD:
        return src.pin_memory().to(dev, non_blocking=True)
    dst = torch.empty(src.shape, dtype=src.dtype, device=dev)
    key = dst.device.index
    with _STAGE_LOCK:
        if key not in _stagers:
            _stagers[key] = _Stager()
        st = _stagers[key]
    st.copy(src, dst)
    return dst


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
        host, ring = _pinned_perm_buffer(count, self.size)
        view = host.numpy()
        for k in range(count):
            view[k] = self.rng.permutation(self.size)
        dev = host.to(self.device, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        with _PERM_LOCK:
            ring.append((host, ev))   # reusable once this copy has completed
        return dev


# pinned staging buffers of PermutationFeeder, reused across draws and fits
# (pinning a fresh buffer per draw costs ~0.3 ms)
_PERM_BUFS: dict = {}
_PERM_LOCK = threading.Lock()


def _pinned_perm_buffer(count: int, size: int):
    with _PERM_LOCK:
        ring = _PERM_BUFS.setdefault((count, size), [])
        for i, (buf, ev) in enumerate(ring):
            if ev.query():
                ring.pop(i)
                return buf, ring
        if len(ring) >= 8:   # all in flight: wait for the oldest
            buf, ev = ring.pop(0)
            ev.synchronize()
            return buf, ring
    return torch.empty((count, size), dtype=torch.int64).pin_memory(), ring
