"""B200-native RAC-MBADMM sweep: drop-in for racml's fit / train / solve hot path.

The re-export surface mirrors the reference package (`racml/__init__.py:3-67`) for
everything on or around the sweep.  The reference's
spectral certificates, LIBSVM I/O, CLI, grid search and model files are out of scope
(SURVEY.md §2 / DESIGN.md §9) and are not exported.

Importing the package does not need a GPU; every solver entry point raises (no CPU
fallback) when the sm_100a library or a B200 is missing.
"""

from .problems import (
    Mode,
    QpProblem,
    SolveResult,
    SolverConfig,
    Status,
    ValidationReport,
    chunk_indices,
    validate_problem,
)
from .engine import (
    BlockDefinitenessError,
    BlockSystem,
    ResidualPair,
    assemble_block_system,
    compute_residuals,
    dual_update,
    run_sweep,
    solve,
    solve_block,
)
from .elastic_net import (
    ElasticNetModel,
    ElasticNetSpec,
    consensus_fit,
    fit,
    objective,
    soft_threshold,
    z_update,
)
from .svm import (
    DegenerateModelError,
    KernelSpec,
    SvmModel,
    TrainDiagnostics,
    accuracy,
    assemble_kernel_block,
    compute_bias,
    kernel_eval,
    predict,
    train,
)

__version__ = "0.1.0"

__all__ = [
    "Mode", "QpProblem", "SolveResult", "SolverConfig", "Status", "ValidationReport", "chunk_indices",
    "validate_problem", "BlockDefinitenessError", "BlockSystem", "ResidualPair", "assemble_block_system",
    "compute_residuals", "dual_update", "run_sweep", "solve", "solve_block", "ElasticNetModel",
    "ElasticNetSpec", "consensus_fit", "fit", "objective", "soft_threshold", "z_update", "DegenerateModelError", "KernelSpec",
    "SvmModel", "TrainDiagnostics", "accuracy", "assemble_kernel_block", "compute_bias", "kernel_eval",
    "predict", "train",
]
