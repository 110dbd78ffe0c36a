"""Small driver for ncu: a few RAC sweeps of one BASELINE config through the native engine."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_01995_b200 import _device, configs, elastic_net as en
from paper_1907_01995_b200.problems import Mode

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
case = configs.GENERATORS[cfg]()
m, n = case.X.shape
gram = sys.argv[3] if len(sys.argv) > 3 else en.choose_gram_mode(m, n, case.block_size, 1000)
sol = en.EnSolver(m, n, case.block_size, Mode.RAC, case.lam, case.alpha, case.gamma)
if gram == "covariance":
    sol.set_gram_mode("covariance")
# device-resident X (rac_en_set_data): G is formed by one split-K Gram + reduce at the
# first run, so a kernel-filtered ncu capture sees G -> factor -> tiles -> chain in order
sol.set_data(torch.from_numpy(case.X).cuda(), case.y)
perms = _device.PermutationFeeder(np.random.default_rng(0), n, sol.dev).draw(sweeps)
sol.run(perms, None)
torch.cuda.synchronize()
print("ok", gram, sol.progress())
