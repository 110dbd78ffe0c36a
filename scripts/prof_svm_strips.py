"""Small driver for ncu: config-4 SVM train with kernel strips formed on the fly (RAC_SVM_STRIPS=1)."""
import os
import sys

sys.path.insert(0, ".")
os.environ["RAC_SVM_STRIPS"] = "1"
from paper_1907_01995_b200 import configs, svm  # noqa: E402
from paper_1907_01995_b200.problems import Mode, SolverConfig  # noqa: E402

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
case = configs.config4()
cfg = SolverConfig(mode=Mode.RAC, block_size=case.block_size, beta_penalty=case.beta, max_iters=sweeps, seed=0,
                   fixed_iterations=True)
_, d = svm.train(case.X, case.labels, case.C, svm.KernelSpec("linear"), cfg, return_diagnostics=True)
print("ok", d.iterations)
