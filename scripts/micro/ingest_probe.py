"""H2D rate of 16 MB pinned chunks, and the row streamer with a no-op consumer (2 GB)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1907_01995_b200 import _device

h = torch.empty(2 * 1024 * 1024, dtype=torch.float64).pin_memory()
d = torch.empty_like(h, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(50):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print("H2D 16 MB chunks: %.1f GB/s" % (50 * h.numel() * 8 / (time.perf_counter() - t) / 1e9))
X = np.random.default_rng(0).standard_normal((50000, 5000))
for rep in range(3):
    t = time.perf_counter()
    _device.stream_rows(X, 32, lambda r0, rows, chunk: None)
    torch.cuda.synchronize()
    print("stream_rows 2 GB no-op consumer: %.1f GB/s" % (X.nbytes / (time.perf_counter() - t) / 1e9))
