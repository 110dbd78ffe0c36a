"""Phase trace of the lookahead covariance chain (main, helper, worker 0) for one sweep."""
import sys
import ctypes
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import _device, configs, elastic_net as en
from paper_1907_01995_b200.problems import Mode

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
case = configs.GENERATORS[cfg]()
m, n = case.X.shape
s = case.block_size
p = -(-n // s)
sol = en.EnSolver(m, n, s, Mode.RAC, case.lam, case.alpha, case.gamma)
sol.set_gram_mode("covariance")
sol.set_data(case.X, case.y)
rng = np.random.default_rng(0)
sol.run(_device.PermutationFeeder(rng, n, sol.dev).draw(5), None)
torch.cuda.synchronize()
lib = sol.lib
for rep in range(2):
    lib.rac_en_set_timing(sol.h, 2)
    sol.run(_device.PermutationFeeder(rng, n, sol.dev).draw(1), None)
    torch.cuda.synchronize()
    ntr = 16 + 28 * p + s
    tb = (ctypes.c_int64 * ntr)()
    lib.rac_en_trace(sol.h, tb, ntr)
    t = np.array(tb[:], dtype=np.float64)
    t0 = t[0]
    rel = lambda v: (v - t0) / 1e3 if v > 0 else float('nan')
    print(f"--- rep {rep}  (us from main start)")
    print(" step | main: start  A_done  B_done  pushed  x_done | helper: tma_issued base_ok waits_ok tq_done | worker0: poll_ok done")
    for u in range(p):
        mn = [rel(t[1 + 5 * u + i]) for i in range(5)]
        hp = [rel(t[1 + 5 * p + 4 * u + i]) for i in range(4)]
        wk = [rel(t[1 + 9 * p + 2 * u + i]) if t[1 + 9 * p + 2 * u + i] != -1 else -1 for i in range(2)]
        print(f"{u:5d} | " + " ".join(f"{x:7.2f}" for x in mn) + " | " + " ".join(f"{x:7.2f}" for x in hp)
              + " | " + " ".join(f"{x:7.2f}" for x in wk))
    ck = t[16 + 16 * p + s:16 + 24 * p + s].reshape(p, 8)
    d = np.diff(ck, axis=1)
    names = ["A: T1 partials", "bar", "B: v", "bar", "C: P + push", "x-spin", "D: sum + next wait"]
    print("clock64 per step (cycles, mean over steps 3..):", {k: round(float(v), 1) for k, v in zip(names, d[3:].mean(axis=0))})
    print("step-to-step cycles:", np.diff(ck[:, 0])[3:].mean())
    hk = t[16 + 24 * p + s:16 + 28 * p + s].reshape(p, 4)
    print("helper clock64 (cycles, mean u>=3): cp_wait+bar %.0f  T-terms %.0f  bar %.0f" % tuple(np.diff(hk, axis=1)[3:].mean(axis=0)))
lib.rac_en_set_timing(sol.h, 0)
info = (ctypes.c_int32 * 4)()
lib.rac_en_info(sol.h, info)
print("info", list(info))
