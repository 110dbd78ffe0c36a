"""One tensor-core Gram of a BASELINE shape, for ncu (config 2: 10000 x 2000; 3: 50000 x 5000)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_01995_b200 import _native

lib = _native.load()
m, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (10000, 2000)
Xc = torch.randn((n, m), dtype=torch.float64, device="cuda")
G = torch.zeros((n, n), dtype=torch.float64, device="cuda")
for _ in range(2):
    _native.check(lib.rac_gram_covariance(C.c_void_p(Xc.data_ptr()), m, m, n, C.c_void_p(G.data_ptr()), float(m), 1))
torch.cuda.synchronize()
