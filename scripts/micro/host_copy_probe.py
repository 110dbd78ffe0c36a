"""Host copy numpy -> pinned staging buffer: torch copy_ vs threaded memmove (GB/s)."""
import ctypes, os, time
from concurrent.futures import ThreadPoolExecutor
import numpy as np
import torch

src = np.random.default_rng(0).standard_normal(20_000_000)     # 160 MB
chunk = 2 * 1024 * 1024                                         # 16 MB in doubles
pinned = torch.empty(chunk, dtype=torch.float64).pin_memory()
print("torch threads", torch.get_num_threads(), "cpus", os.cpu_count())

def torch_copy():
    for off in range(0, src.size, chunk):
        n = min(chunk, src.size - off)
        pinned[:n].copy_(torch.from_numpy(src[off:off + n]))

pool = ThreadPoolExecutor(16)
def threaded(nt):
    dst = pinned.data_ptr()
    def part(args):
        a, b, base = args
        ctypes.memmove(dst + a * 8, base + a * 8, (b - a) * 8)
    for off in range(0, src.size, chunk):
        n = min(chunk, src.size - off)
        base = src[off:].ctypes.data
        step = (n + nt - 1) // nt
        list(pool.map(part, [(i, min(n, i + step), base) for i in range(0, n, step)]))

for name, fn in [("torch", torch_copy), ("mm4", lambda: threaded(4)), ("mm8", lambda: threaded(8)), ("mm16", lambda: threaded(16)), ("torch", torch_copy)]:
    fn()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {src.nbytes / dt / 1e9:.1f} GB/s")
