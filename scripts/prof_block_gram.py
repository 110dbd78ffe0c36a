"""One block-mode sweep of config 5 (5000 x 100000, s = 500) for ncu of the int8 block Grams."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1907_01995_b200 import _device, configs, elastic_net as en
from paper_1907_01995_b200.problems import Mode

case = configs.GENERATORS[5]()
m, n = case.X.shape
sol = en.EnSolver(m, n, case.block_size, Mode.RAC, case.lam, case.alpha, case.gamma)
sol.set_data(torch.from_numpy(case.X).cuda(), case.y)
feeder = _device.PermutationFeeder(np.random.default_rng(0), n, sol.dev)
sol.run(feeder.draw(2), None)
torch.cuda.synchronize()
