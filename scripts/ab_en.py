"""A/B timing of one BASELINE EN config under several environment settings (one process).

usage: ab_en.py <config> <sweeps> [ENV=val[,ENV=val...]] ...   ('-' = no overrides)
Each setting creates a fresh solver (the RAC_* switches are read at context creation),
times <sweeps> pipelined sweeps with CUDA events, then the per-stage breakdown."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1907_01995_b200 import _device, configs, elastic_net as en
from paper_1907_01995_b200.problems import Mode

cfg = int(sys.argv[1])
K = int(sys.argv[2])
settings = sys.argv[3:] or ['-']
case = configs.GENERATORS[cfg]()
m, n = case.X.shape
s = case.block_size
gram = en.choose_gram_mode(m, n, s, 1000)
Xd = torch.from_numpy(case.X).cuda()
for st in settings:
    envs = {} if st == '-' else dict(kv.split('=') for kv in st.split(','))
    old = {k: os.environ.get(k) for k in envs}
    os.environ.update(envs)
    try:
        sol = en.EnSolver(m, n, s, Mode.RAC, case.lam, case.alpha, case.gamma)
        if gram == "covariance":
            sol.set_gram_mode("covariance")
        sol.set_data(Xd, case.y)
        rng = np.random.default_rng(0)
        feeder = _device.PermutationFeeder(rng, n, sol.dev)
        sol.run(feeder.draw(4), None)
        torch.cuda.synchronize()
        best = 1e9
        for rep in range(3):
            perms = feeder.draw(K)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if gram == "covariance":
                sol.set_gram_mode("covariance")
            sol.run(perms, None)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / K)
        lib = sol.lib
        lib.rac_en_set_timing(sol.h, 1)
        sol.run(feeder.draw(K), None)
        stage = (ctypes.c_double * 4)()
        nt = ctypes.c_int32()
        lib.rac_en_timing(sol.h, stage, nt)
        lib.rac_en_set_timing(sol.h, 0)
        stages = [float(v) / max(nt.value, 1) for v in stage]
        st_, sw, res = sol.progress()[:3] if len(sol.progress()) >= 3 else (0, 0, 0)
        print(f"cfg{cfg} {st:40s} ms/sweep {best:8.4f}  sweeps/s {1e3 / best:9.1f}  stages[asm,gram,factor,chain] "
              + " ".join(f"{v:.4f}" for v in stages) + f"  progress {sol.progress()}", flush=True)
        sol.close()
        del sol
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
