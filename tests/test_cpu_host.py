"""CPU-only tests: contract types, validation, the C-ABI library surface, replicas over gloo."""

import os
import re
import socket
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rac_b200.h")


# ---------------------------------------------------------------- C ABI
def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rac_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    fns = header_functions()
    for name in ("rac_chunk_sort", "rac_en_create", "rac_en_run", "rac_qp_create", "rac_qp_run",
                 "rac_svm_build_q", "rac_box_block_min", "rac_gram_inverse"):
        assert name in fns


def test_library_exports_every_header_symbol():
    from paper_1907_01995_b200 import _native
    lib = _native.load()
    assert _native.MISSING == []
    for name in header_functions():
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (rac_[a-z0-9_]+)", out))
    assert set(header_functions()) <= exported


def test_library_is_sm100a():
    from paper_1907_01995_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_version_and_no_device_error():
    from paper_1907_01995_b200 import _native
    lib = _native.load()
    assert b"sm_100a" in lib.rac_version()
    import torch
    if not torch.cuda.is_available():
        assert lib.rac_device_check(0) != 0
        assert lib.rac_last_error()


def test_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1907_01995_b200 import elastic_net as en
    with pytest.raises(RuntimeError):
        en.fit(np.eye(3), np.ones(3), en.ElasticNetSpec(lam=0.1, alpha=1.0, block_size=1, iters=1))


def test_argument_errors_cross_abi_as_codes():
    from paper_1907_01995_b200 import _native
    lib = _native.load()
    assert lib.rac_chunk_sort(None, 10, 3, 1, None, None) == _native.RAC_ERR_ARG
    assert b"bad arguments" in lib.rac_last_error()


# ---------------------------------------------------------------- contract types
def test_solver_config_validation_messages():
    from paper_1907_01995_b200.problems import SolverConfig
    with pytest.raises(ValueError, match="beta_penalty"):
        SolverConfig(beta_penalty=0).validate(5)
    with pytest.raises(ValueError, match="block_size"):
        SolverConfig(block_size=6).validate(5)
    with pytest.raises(ValueError, match="tolerances"):
        SolverConfig(tol_primal=0).validate(500)
    with pytest.raises(ValueError, match="max_iters"):
        SolverConfig(max_iters=0).validate(500)
    SolverConfig().validate(500)


def test_validate_problem_reports_all_issues():
    from paper_1907_01995_b200.problems import QpProblem, validate_problem
    p = QpProblem(c=np.array([1.0, np.nan]), H=np.array([[1.0, 2.0], [0.0, 1.0]]), A=np.ones((1, 3)),
                  lower=np.array([1.0, 0.0]), upper=np.array([0.0, 1.0]))
    rep = validate_problem(p)
    assert not rep.ok and not bool(rep)
    text = "; ".join(rep.issues)
    for frag in ("not symmetric", "expected 2 columns", "b: required", "c: contains non-finite",
                 "lower > upper"):
        assert frag in text, frag


def test_chunk_indices_twin_matches_oracle():
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200.problems import chunk_indices
    rng = np.random.default_rng(0)
    perm = rng.permutation(103)
    got = chunk_indices(perm, 10)
    want = ro.sorted_chunks(perm, 10)
    assert len(got) == len(want) == 11
    for a, b in zip(got, want):
        assert list(a) == list(b)


def test_elastic_net_spec_validation():
    from paper_1907_01995_b200.elastic_net import ElasticNetSpec
    from paper_1907_01995_b200.problems import Mode
    for kw, frag in [(dict(lam=-1, alpha=0.5), "lam"), (dict(lam=1, alpha=2), "alpha"),
                     (dict(lam=1, alpha=0.5, gamma=0), "gamma"), (dict(lam=1, alpha=0.5, block_size=0), "block_size"),
                     (dict(lam=1, alpha=0.5, iters=0), "iters"),
                     (dict(lam=1, alpha=0.5, mode=Mode.CYCLIC), "mode")]:
        with pytest.raises(ValueError, match=frag):
            ElasticNetSpec(**kw).validate()


def test_resolve_gamma_density_rule():
    import scipy.sparse as sp
    from paper_1907_01995_b200.elastic_net import ElasticNetSpec, resolve_gamma
    spec = ElasticNetSpec(lam=0.4, alpha=1.0)
    assert resolve_gamma(spec, np.ones((10, 10))) == pytest.approx(0.04)
    assert resolve_gamma(spec, sp.csc_matrix((1000, 1000))) == pytest.approx(0.4)
    assert resolve_gamma(ElasticNetSpec(lam=0.0, alpha=1.0), np.ones((2, 2))) == 1.0
    assert resolve_gamma(ElasticNetSpec(lam=1.0, alpha=1.0, gamma=2.5), np.eye(3)) == 2.5


def test_soft_threshold_and_z_update_host_twins(golden):
    from paper_1907_01995_b200 import elastic_net as en
    g = golden("block_prox")
    assert en.soft_threshold(3.0, 1.0) == -2.0
    assert en.soft_threshold(-3.0, 1.0) == 2.0
    assert en.soft_threshold(0.5, 1.0) == 0.0
    with pytest.raises(ValueError):
        en.soft_threshold(1.0, -0.1)
    assert np.array_equal(en.z_update(g["prox_beta"], g["prox_xi"], 0.7, 0.4, 0.3), g["prox_z"])
    with pytest.raises(ValueError):
        en.z_update(1.0, 1.0, 0.0, 1.0, 0.5)


def test_svm_defaults():
    from paper_1907_01995_b200 import svm
    assert svm.default_block_size(500) == 100
    assert svm.default_block_size(50_000) == 500
    assert svm.default_block_size(200_000) == 1000
    assert svm.default_config(1000, block_size=100).beta_penalty == pytest.approx(1.0)
    with pytest.raises(ValueError):
        svm.KernelSpec("poly").validate()
    with pytest.raises(ValueError):
        svm.KernelSpec("gaussian", 0.0).validate()


def test_config_generators_shapes():
    from paper_1907_01995_b200 import configs
    c = configs.config2(scale=0.05)
    assert c.X.shape == (500, 100)
    assert np.allclose(np.linalg.norm(c.X / np.sqrt(500), axis=0), 1.0)
    c4 = configs.config4(scale=0.01)
    assert set(np.unique(c4.labels)) == {-1.0, 1.0}


# ---------------------------------------------------------------- replicas over gloo (world 2)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _replica_worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import rac_oracle as ro
    from paper_1907_01995_b200 import replicas
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cells = [(lam, alpha) for lam in (0.01, 0.1, 1.0) for alpha in (0.5, 1.0)]
    mine = replicas.shard(cells, rank, world)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((40, 12))
    y = rng.standard_normal(40)
    local = [(c, ro.en_fit(X, y, c[0], c[1], 1.0, 4, 5, seed=0)["iterations"]) for c in mine]
    allres = replicas.gather_results(local)
    tmax = replicas.max_over_ranks(float(rank + 1))
    q.put((rank, sorted(c for c, _ in allres), tmax))
    dist.destroy_process_group()


def test_replica_grid_over_gloo_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cells = sorted((lam, alpha) for lam in (0.01, 0.1, 1.0) for alpha in (0.5, 1.0))
    for rank, got, tmax in out:
        assert got == cells          # every cell solved exactly once across ranks
        assert tmax == 2.0           # max over ranks


def test_shard_covers_once():
    from paper_1907_01995_b200 import replicas
    cells = list(range(11))
    parts = [replicas.shard(cells, r, 3) for r in range(3)]
    assert sorted(sum(parts, [])) == cells
    with pytest.raises(ValueError):
        replicas.shard(cells, 3, 3)


def test_fit_context_pool_reuse_env_keys_and_eviction(monkeypatch):
    """fit()'s native-context pool (host logic, no GPU): a released context of the same
    shape is reset and reused; RAC_* variant switches are part of the key; a failed fit's
    context is closed, not pooled; at most _POOL_MAX idle contexts stay (LRU)."""
    from paper_1907_01995_b200 import elastic_net as en
    from paper_1907_01995_b200.problems import Mode
    events = []

    class FakeSolver:
        def __init__(self, m, n, s, mode, lam, alpha, gamma, device=0):
            self.m = m
            events.append(("new", m))

        def reset(self, lam, alpha, gamma):
            events.append(("reset", self.m))

        def close(self):
            events.append(("close", self.m))

    monkeypatch.setattr(en, "EnSolver", FakeSolver)
    monkeypatch.setattr(en._device, "stream_handle", lambda *a, **k: 0)
    for k in [k for k in list(__import__("os").environ) if k.startswith("RAC_")]:
        monkeypatch.delenv(k)
    en._POOL.clear()
    k1, s1 = en._acquire_solver(10, 20, 5, Mode.RAC, 0.1, 1.0, 1.0, 0)
    en._release_solver(k1, s1, True)
    k2, s2 = en._acquire_solver(10, 20, 5, Mode.RAC, 0.2, 1.0, 1.0, 0)
    assert s2 is s1 and events[-1] == ("reset", 10)
    en._release_solver(k2, s2, True)
    monkeypatch.setenv("RAC_CLA_D", "2")
    k3, s3 = en._acquire_solver(10, 20, 5, Mode.RAC, 0.2, 1.0, 1.0, 0)
    assert s3 is not s1 and events[-1] == ("new", 10)
    en._release_solver(k3, s3, False)
    assert events[-1] == ("close", 10)
    monkeypatch.delenv("RAC_CLA_D")
    for i in range(6):
        k, sv = en._acquire_solver(100 + i, 20, 5, Mode.RAC, 0.1, 1.0, 1.0, 0)
        en._release_solver(k, sv, True)
    assert len(en._POOL) == en._POOL_MAX
    assert ("close", 10) in events and ("close", 100) in events   # least recently used first
    en._POOL.clear()


def test_package_reexports_reference_surface():
    """The racml re-export names that belong to the sweep (racml/__init__.py:3-67, SURVEY §8(a)
    a13) are importable from the package root; spectral / data_io / CLI are out of scope."""
    import paper_1907_01995_b200 as rac
    for name in ("Mode", "QpProblem", "SolveResult", "SolverConfig", "Status", "ValidationReport",
                 "validate_problem", "BlockDefinitenessError", "BlockSystem", "ResidualPair",
                 "assemble_block_system", "compute_residuals", "dual_update", "run_sweep", "solve", "solve_block",
                 "ElasticNetModel", "ElasticNetSpec", "fit", "soft_threshold", "z_update", "KernelSpec", "SvmModel",
                 "accuracy", "assemble_kernel_block", "compute_bias", "kernel_eval", "predict", "train"):
        assert hasattr(rac, name), name
    bs = rac.BlockSystem(np.eye(2), np.ones(2), np.array([-np.inf, 0.0]), np.array([np.inf, np.inf]))
    assert bs.bounded is True
    assert rac.BlockSystem(np.eye(1), np.ones(1), np.array([-np.inf]), np.array([np.inf])).bounded is False
    rp = rac.ResidualPair(primal=1.0, dual=2.0, primal_l1=3.0)
    with pytest.raises(Exception):
        rp.primal = 0.0          # frozen like the reference's


def test_helpers_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_1907_01995_b200 as rac
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rac.solve_block(rac.BlockSystem(np.eye(1), np.ones(1), np.zeros(1), np.ones(1)))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rac.assemble_kernel_block(np.eye(3), np.ones(3), [0, 1], rac.KernelSpec("linear"))
