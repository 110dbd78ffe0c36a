"""Is cudaHostRegister + direct DMA of a 160 MB numpy array faster than pinned staging?"""
import ctypes, time
import numpy as np
import torch
cudart = ctypes.CDLL("libcudart.so")
X = np.random.default_rng(0).standard_normal((10000, 2000))
dev = torch.empty(X.shape, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for rep in range(4):
    t0 = time.perf_counter()
    rc = cudart.cudaHostRegister(ctypes.c_void_p(X.ctypes.data), ctypes.c_size_t(X.nbytes), 0)
    t1 = time.perf_counter()
    dev.copy_(torch.from_numpy(X), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cudart.cudaHostUnregister(ctypes.c_void_p(X.ctypes.data))
    t3 = time.perf_counter()
    print(f"rc={rc} register {1e3*(t1-t0):.2f} ms  DMA {1e3*(t2-t1):.2f} ms ({X.nbytes/(t2-t1)/1e9:.1f} GB/s)  unregister {1e3*(t3-t2):.2f} ms  total {1e3*(t3-t0):.2f}")
