"""Benchmark: RAC-ADMM sweeps/sec and time to 1e-6 on one B200, beside the CPU reference path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C] [--only]

A "step" is one RAC sweep: one pass of the Gauss-Seidel chain over all p blocks,
including that sweep's block assembly, block Grams and factorizations.

The headline workload is BASELINE.json's largest single-GPU configuration, config 5
(HD-LASSO, D 5000 x 100000, s = 500; BASELINE's metric names no config).  The same
JSON line carries a `configs` object with every BASELINE config (1-5): device
sweeps/s, end-to-end sweeps/s through the public API, time to tolerance (device and
end to end), the roofline of its dominant kernel and the CPU port beside it.
`--only` skips the other configs.

Multi-GPU: the sweep is a sequential Gauss-Seidel chain, so N > 1 runs N independent
replicas (one per GPU, `scaling: weak`, max-over-ranks device time).  Without
torchrun, `--gpus N` re-launches itself under torch.distributed.run with N ranks.
"""

from __future__ import annotations

import argparse
import gc
import glob
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HEADLINE = 5
HBM_FALLBACK_GBS = 6650.0
INT8_DENSE_TOPS_NOMINAL = 4500.0
METRIC = "rac_admm_sweeps_per_sec"
DATA = "synthetic (SURVEY.md §8(d) seed-0 recipe; BASELINE names no dataset)"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxes.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ------------------------------------------------------------------ distributed
def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` without torchrun: run this script as N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


def dist_setup(backend: str):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def dist_max(value: float, world: int, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ workloads
def make_case(cfg: int):
    from paper_1907_01995_b200 import configs
    return configs.GENERATORS[cfg]()


def config_dict(cfg: int, case, steps: int, world: int) -> dict:
    """The `config` object of a line (identical in both arms, so the driver can pair them)."""
    if cfg == 4:
        N, d = case.X.shape
        s = case.block_size
        return {"workload": case.name, "N": N, "d": d, "block_size": s, "blocks": -(-N // s), "mode": "rac",
                "l2": "inputs larger than L2 (Q = %.1f GB)" % (8 * N * N / 1e9),
                "parallelism": f"replicas x{world}"}
    from paper_1907_01995_b200 import elastic_net as en
    m, n = case.X.shape
    s = min(case.block_size, n)
    return {"workload": case.name, "m": m, "n": n, "block_size": s, "blocks": -(-n // s), "mode": "rac",
            "gram_mode": en.choose_gram_mode(m, n, s, steps),
            "l2": ("inputs larger than L2 (D = %.0f MB)" % (8 * m * n / 1e6)) if 8 * m * n > 126e6
            else "D fits in L2 (no flush)",
            "parallelism": f"replicas x{world}"}


def traffic_table() -> dict:
    """DRAM bytes per launch from committed ncu --set full captures (profiles/*traffic*.json),
    keyed "<workload>:<kernel>"."""
    out = {}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*traffic*.json"))):
        try:
            with open(path) as f:
                out.update(json.load(f))
        except (OSError, ValueError):
            pass
    return out


def block_grams_int8(s: int, p: int, sms: int = 148) -> bool:
    """Mirror of the context's rule (csrc/en.cu rac_en_create): block-mode Grams run on the
    int8 tensor cores when a sweep's 128 x 128 tiles fill the SMs four times."""
    mode = int(os.environ.get("RAC_BG_I8", "1"))
    jt = (s + 127) // 128
    return mode == 2 or (mode == 1 and s >= 128 and p * jt * (jt + 1) // 2 >= 4 * sms)


def fp64_peak_tflops(torch) -> float:
    """Measured cuBLAS DGEMM (8192^3 fp64) on this device, best of 5 — FP64 roofline denominator."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn_like(a)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = math.inf
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * 8192 ** 3 / (best * 1e-3) / 1e12


def int8_peak_tops(torch, peaks: dict) -> dict:
    """INT8 tensor denominator: the larger of a measured cuBLASLt int8 GEMM (torch._int_mm,
    8192^3, best of 5) and 2 x the driver-measured bf16 burst (dense INT8 issues at twice the
    bf16 rate on sm_100).  The larger one is the conservative denominator."""
    meas = None
    try:
        a = torch.randint(-64, 64, (8192, 8192), dtype=torch.int8, device="cuda")
        b = torch.randint(-64, 64, (8192, 8192), dtype=torch.int8, device="cuda")
        torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = math.inf
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        meas = 2.0 * 8192 ** 3 / (best * 1e-3) / 1e12
        del a, b
    except Exception:   # noqa: BLE001 — no int8 GEMM in this torch build
        meas = None
    derived = 2.0 * peaks["bf16_tflops"] if "bf16_tflops" in peaks else None
    cands = [v for v in (meas, derived) if v]
    peak = max(cands) if cands else INT8_DENSE_TOPS_NOMINAL
    return {"peak": peak, "cublaslt_int8_tops": meas, "two_x_bf16_measured": derived,
            "nominal": INT8_DENSE_TOPS_NOMINAL,
            "source": "max(measured torch._int_mm 8192^3, 2 x MEASURED_PEAKS bf16_tflops)" if cands else
                      "nominal (no measurement)"}


def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        blas = [i["num_threads"] for i in info if i.get("internal_api") in ("openblas", "mkl", "blis")]
        if blas:
            return int(max(blas))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def cpu_sweep_times(cfg: int, case, sweeps: int) -> list[float]:
    """Per-sweep wall times of the oracle port (numpy restatement of racml fit / train) over
    `sweeps` consecutive sweeps of ONE call; the setup (c = -X'y/m) is outside every sweep."""
    from oracle import rac_oracle as ro
    stamps = [time.perf_counter()]
    if cfg == 4:
        ro.svm_train(case.X, case.labels, case.C, "linear", block_size=case.block_size, beta=case.beta,
                     max_iters=sweeps, seed=case.seed, fixed_iterations=True,
                     on_sweep=lambda *a: stamps.append(time.perf_counter()))
    else:
        def first(*a):
            stamps.append(time.perf_counter())
        ro.en_fit(case.X, case.y, case.lam, case.alpha, case.gamma, case.block_size, sweeps,
                  seed=case.seed, tol=None, on_sweep=first)
    return list(np.diff(stamps[1:])) if len(stamps) > 2 else []


class _SampleDone(Exception):
    pass


def cpu_baseline(cfg: int, case, budget_s: float = 8.0) -> dict:
    """Bounded sample of the oracle port on the host cores: consecutive sweeps of ONE call,
    stopped once `budget_s` has elapsed (at least 2 sweeps); the first sweep carries the
    call's setup and is not counted."""
    from oracle import rac_oracle as ro
    stamps = []
    t0 = time.perf_counter()

    def cb(*a):
        stamps.append(time.perf_counter())
        if len(stamps) >= 3 and stamps[-1] - t0 >= budget_s:
            raise _SampleDone()

    try:
        if cfg == 4:
            ro.svm_train(case.X, case.labels, case.C, "linear", block_size=case.block_size, beta=case.beta,
                         max_iters=40, seed=case.seed, fixed_iterations=True, on_sweep=cb)
        else:
            ro.en_fit(case.X, case.y, case.lam, case.alpha, case.gamma, case.block_size, 40,
                      seed=case.seed, on_sweep=cb)
    except _SampleDone:
        pass
    total = time.perf_counter() - t0
    fn = "svm_train" if cfg == 4 else "en_fit"
    rate = (len(stamps) - 1) / (stamps[-1] - stamps[0])
    return {"value": rate, "unit": "sweeps/s", "cores": cpu_threads(), "kind": "port",
            "sample": f"sweeps 2..{len(stamps)} of one oracle/rac_oracle.{fn} call on {case.name} "
                      f"({total:.1f} s; the first sweep, incl. setup, excluded)"}


# ------------------------------------------------------------------ reference arm
def run_reference(args) -> int:
    """--impl reference: the reference's CPU algorithm (the oracle port: same numpy/scipy
    calls as racml) on the host cores, K consecutive sweeps of the headline config in ONE
    call, W warm-up sweeps before them in the same call (setup outside the timer)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    case = make_case(args.config)
    K, W = args.steps, args.warmup
    t0 = time.perf_counter()
    times = cpu_sweep_times(args.config, case, W + K)
    total = time.perf_counter() - t0
    timed = times[W - 1:W - 1 + K] if W >= 1 else times[:K]
    if len(timed) < K:      # W = 0: the first sweep carries the setup; use what was timed
        timed = times[-K:]
    sec = float(sum(timed))
    rate = len(timed) / sec
    fn = "svm_train" if args.config == 4 else "en_fit"
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "sweeps/s", "n_gpus": 0,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * sec / len(timed), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": config_dict(args.config, case, K, world),
        "cpu_baseline": {"value": rate, "unit": "sweeps/s", "cores": cpu_threads(), "kind": "port",
                         "sample": f"sweeps {W + 1}..{W + K} of one oracle/rac_oracle.{fn} call "
                                   f"({W + K} sweeps, {total:.1f} s incl. setup)"},
        "e2e": {"value": rate, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ roofline
def en_roofline(stages, m, n, s, p, gram_mode, variant, hbm, fp64, i8, workload, prep_batch=1, slices=8) -> dict:
    """Roofline entry for the dominant stage of an EN sweep (per-unit figures: SURVEY.md §8(d),
    DESIGN.md §4).  `stages` are per-sweep times measured with CUDA events; in covariance mode
    the block systems of `prep_batch` sweeps are prepared by one launch that overlaps the chain,
    so the stage that bounds a sweep is picked on factor / prep_batch."""
    eff = dict(stages)
    eff["factor"] = stages.get("factor", 0.0) / max(1, prep_batch)
    eff.pop("assembly", None)
    dom = max(eff, key=eff.get)
    roof = en_stage_roofline(dom, stages, m, n, s, p, gram_mode, variant, hbm, fp64, i8, slices)
    roof["traffic"] = traffic_table().get(f"{workload}:{roof['kernel'].split()[0]}")
    # every stage against its own roof (the headline entry above is the stage that bounds a sweep)
    roof["all_stages"] = [
        {k: v for k, v in en_stage_roofline(st, stages, m, n, s, p, gram_mode, variant, hbm, fp64, i8, slices).items()
         if k in ("stage", "kernel", "bound", "achieved", "peak", "unit", "frac")}
        | {"ms_per_sweep": stages[st]}
        for st in ("gram", "factor", "chain")
        if stages.get(st, 0.0) > 0.0 and not (st == "gram" and gram_mode == "covariance")]   # G: once per fit
    return roof


def en_stage_roofline(dom, stages, m, n, s, p, gram_mode, variant, hbm, fp64, i8, slices) -> dict:
    """One stage's kernel against the roof that bounds it (algorithmic work per sweep ÷ the stage's
    measured time per sweep)."""
    sec = stages[dom] * 1e-3
    if dom == "chain":
        if gram_mode == "covariance":
            kern = "en_cla_kernel" if variant == "covariance-lookahead" else "en_cov_kernel"
            byts = 8.0 * n * n + 8.0 * p * s * s
            desc = "rows of G read once (8 n^2) + block inverses (8 p s^2) per launch"
        else:
            kern = "en_chain_res_kernel" if variant == "resident-cluster" else "en_chain_kernel"
            byts = 8.0 * m * n + 8.0 * p * s * s
            desc = "D read once (8 m n; a block's second use hits L2) + block inverses (8 p s^2) per launch"
        achieved = byts / sec / 1e9
        roof = {"kernel": kern, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "algorithmic": desc}
    elif dom == "gram" and gram_mode == "blocks" and block_grams_int8(s, p) and slices > 0:
        jt = (s + 127) // 128
        prods = slices * (slices + 1) // 2        # slice pairs s + t <= S + 1
        ops = 2.0 * prods * p * (jt * (jt + 1) // 2) * 128 * 128 * ((m + 31) // 32 * 32)
        achieved = ops / sec / 1e12
        roof = {"kernel": "gram_i8_kernel (tcgen05 kind::i8, + digit slicing)", "bound": "tensor",
                "achieved": achieved, "peak": i8["peak"], "unit": "TOPS (int8)", "frac": achieved / i8["peak"],
                "peak_source": i8["source"],
                "slices": slices,
                "algorithmic": f"{prods} int8 digit-slice products ({slices} slices) x 2*128*128*K per upper "
                               "tile of each of the p blocks per sweep (FP64-level block Grams)",
                "fp64_equivalent": {"achieved_tflops": float(m) * n * (s + 1) / sec / 1e12, "peak": fp64,
                                    "frac": float(m) * n * (s + 1) / sec / 1e12 / fp64,
                                    "algorithmic": "m*n*(s+1) flop per sweep (symmetric SYRK of all p blocks)"}}
    elif dom == "gram":
        achieved = float(m) * n * (s + 1) / sec / 1e12
        roof = {"kernel": "gram_kernel", "bound": "tensor", "achieved": achieved, "peak": fp64,
                "unit": "TFLOP/s", "frac": achieved / fp64,
                "algorithmic": "m*n*(s+1) flop per launch (symmetric SYRK of all p blocks)"}
    else:
        achieved = 2.0 * p * float(s) ** 3 / sec / 1e12
        roof = {"kernel": "factor_kernel" if s <= 236 else "large_*_kernel (blocked inverse)",
                "bound": "tensor", "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
                "frac": achieved / fp64, "algorithmic": "2 s^3 flop per block inverse x p blocks per sweep"}
    roof["stage"] = dom
    return roof


# ------------------------------------------------------------------ B200 arm: elastic net
def _ev():
    import torch
    return torch.cuda.Event(enable_timing=True)


def measure_en(cfg, case, args, world, rank, local, peaks, fp64, i8, headline: bool) -> dict:
    import torch
    from paper_1907_01995_b200 import _device, elastic_net as en
    from paper_1907_01995_b200.problems import Mode

    dev = torch.device("cuda", local)
    m, n = case.X.shape
    s = min(case.block_size, n)
    p = -(-n // s)
    K, W = args.steps, args.warmup
    gram_mode = args.gram if args.gram != "auto" else en.choose_gram_mode(m, n, s, K)
    out: dict = {}

    # ---------------- device-resident throughput (fixed sweeps, every sweep does full work)
    solver = en.EnSolver(m, n, s, Mode.RAC, case.lam, case.alpha, case.gamma, device=local)
    if gram_mode == "covariance":
        solver.set_gram_mode("covariance")
    solver.set_data(case.X, case.y)
    rng = np.random.default_rng(case.seed)
    perms = _device.PermutationFeeder(rng, n, dev).draw(W + K)
    solver.run(perms[:W], None)
    gc.collect()
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if headline else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    dist_barrier(world)
    torch.cuda.synchronize()
    e0, e1 = _ev(), _ev()
    l0 = solver.lib.rac_launch_count()
    e0.record()
    if gram_mode == "covariance":
        solver.set_gram_mode("covariance")   # G = X'X/m is re-formed INSIDE the timed region
    solver.run(perms[W:W + K], None)
    e1.record()
    launches = solver.lib.rac_launch_count() - l0
    torch.cuda.synchronize()
    dist_barrier(world)
    if clocks:
        out["clocks"] = clocks.stop()
    ms = dist_max(e0.elapsed_time(e1), world, dev)
    out.update({"value": world * K / (ms * 1e-3), "ms_per_step": ms / K, "gpu_launches": int(launches),
                "gram_mode": gram_mode})

    # ---------------- per-stage breakdown (separate sweeps, CUDA events between stages)
    lib = solver.lib
    lib.rac_en_set_timing(solver.h, 1)
    solver.run(_device.PermutationFeeder(rng, n, dev).draw(K), None)
    stage = (np.ctypeslib.ctypes.c_double * 4)()
    nt = np.ctypeslib.ctypes.c_int32()
    lib.rac_en_timing(solver.h, stage, nt)
    stages = {k: float(v) / max(nt.value, 1) for k, v in zip(("assembly", "gram", "factor", "chain"), stage)}
    out["stage_ms_per_sweep"] = stages
    # int8 block Grams: the gram stage is two kernels (digit slicing, then the tcgen05 GEMM)
    sl_ms = np.ctypeslib.ctypes.c_double(0.0)
    lib.rac_en_timing_slicing(solver.h, np.ctypeslib.ctypes.byref(sl_ms))
    slice_ms = sl_ms.value / max(nt.value, 1)
    if slice_ms > 0.0:
        out["gram_stage_split_ms"] = {"i8_slice_kernel": slice_ms, "gram_i8_kernel": stages["gram"] - slice_ms}
    # chain phase trace (CTA 0 %globaltimer at each phase boundary of one sweep)
    lib.rac_en_set_timing(solver.h, 2)
    solver.run(_device.PermutationFeeder(rng, n, dev).draw(1), None)
    torch.cuda.synchronize()
    ntr = 16 + 20 * p + s
    tbuf = (np.ctypeslib.ctypes.c_int64 * ntr)()
    lib.rac_en_trace(solver.h, tbuf, ntr)
    info = (np.ctypeslib.ctypes.c_int32 * 4)()
    lib.rac_en_info(solver.h, info)
    sl = np.ctypeslib.ctypes.c_int32(0)
    lib.rac_en_gram_slices(solver.h, np.ctypeslib.ctypes.byref(sl))
    slices = int(sl.value)          # digit slices of the int8 Grams (0: FP64 DMMA tiles)
    labels = (("delta_sum_next_wait", "t1_term", "v", "partials_push", "exchange_wait")
              if info[0] == 3 else
              ("cluster_sync", "cluster_reduce", "grid_barrier", "commit", "rhs_loads", "solve_wait", "rhs",
               "delta+cluster_sync", "tile_wait",
               "row_pass1", "row_sync1", "row_pass2", "row_pass3", "issue_next")
              if info[0] == 1 else
              ("barrier1", "S1_reduce", "barrier2", "S2_solve", "barrier3", "row_phase") if info[0] == 0 else
              ("phase_a_q_update", "cluster_sync1", "prefetch_wait", "v_gather", "delta_commit", "cluster_sync2",
               "delta_gather"))
    nl = len(labels)
    variant = {0: "streaming", 1: "resident-cluster", 2: "covariance-cluster",
               3: "covariance-lookahead"}[int(info[0])]
    chain_trace = {"variant": variant, "ctas": int(info[1]), "gram_mode": gram_mode}
    pro = {0: 2, 1: 5, 2: 1, 3: 1}[int(info[0])]   # stamps before the first block
    if info[0] == 3:
        chain_trace.update({"prep_batch_sweeps": int(info[2]), "lookahead_depth": int(info[3])})
    else:
        chain_trace.update({"rows_per_chunk": int(info[2]), "chunks_per_cta": int(info[3])})
    tv = np.array(tbuf[:pro + nl * p], dtype=np.float64) / 1e3   # us
    if tv[0] > 0:
        ph = np.diff(tv[pro - 1:]).reshape(p, nl)
        chain_trace.update({"first_phase_us": float(tv[pro - 1] - tv[0]),
                            "per_block_us": {k: float(v) for k, v in zip(labels, ph.mean(axis=0))}})
        if info[0] == 0 and int(info[2]) == 0 and p > 1:
            # one-tile row phase split: (a) r += X_prev delta, tile load, (c) t = r - X_next beta_next,
            # (d) partials X_next' t (CTA 0 stamps; the last block has no next tile)
            rt = np.array(tbuf[16 + 16 * p + s:16 + 20 * p + s], dtype=np.float64).reshape(p, 4)[:p - 1] / 1e3
            start = tv[pro + 6 * np.arange(p - 1) + 4]
            d = np.diff(np.c_[start, rt], axis=1)
            chain_trace["row_phase_split_us"] = {k: float(v) for k, v in
                                                 zip(("a_r_update", "tile_load", "c_t", "d_partials"), d.mean(axis=0))}
    if s <= 236:
        # factor kernel, block 0: assembly, then per 8-pivot step [panel copy, 8x8 sweep, CW, update]
        f0 = 8 + 16 * p
        nst = (s + 7) // 8
        fv = np.array(tbuf[f0:f0 + 2 + 4 * nst], dtype=np.float64) / 1e3
        if fv[0] > 0 and fv[-1] > 0:
            steps = np.diff(np.r_[fv[1], fv[2:]]).reshape(nst, 4)
            chain_trace["factor_block0_us"] = {
                "assembly": float(fv[1] - fv[0]), "steps": int(nst),
                "per_step": {k: float(v) for k, v in zip(("panel", "diag_sweep", "cw", "update"),
                                                         steps.mean(axis=0))}}
    lib.rac_en_set_timing(solver.h, 0)
    out["chain_trace"] = chain_trace
    solver.close()
    del perms

    # ---------------- time to tolerance, device: X resident in HBM before the timer; the
    # timer covers set_data (transpose into the column-major layout and, in covariance mode,
    # the once-per-fit G = X'X/m) and every sweep, driven like fit() with a tolerance
    ttt = None
    if case.tol is not None:
        tol_gm = en.choose_gram_mode(m, n, s, case.iters) if args.gram == "auto" else args.gram
        Xd = torch.from_numpy(np.ascontiguousarray(case.X)).to(dev)
        yd = torch.from_numpy(np.ascontiguousarray(case.y)).to(dev)
        sol2 = en.EnSolver(m, n, s, Mode.RAC, case.lam, case.alpha, case.gamma, device=local)
        if tol_gm == "covariance":
            sol2.set_gram_mode("covariance")    # reserves G's memory; G itself is formed in the timer
        rng2 = np.random.default_rng(case.seed)
        feeder = _device.PermutationFeeder(rng2, n, dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol2.set_data(Xd, yd)
        sol2.run(feeder.draw(min(16, case.iters)), case.tol)
        done = min(16, case.iters)
        while True:
            lag = 0
            if done < case.iters:
                k = min(16, case.iters - done)
                sol2.run(feeder.draw(k), case.tol)
                done += k
                lag = 1
            _, conv, failed = sol2.poll(lag)
            if failed >= 0 or conv or lag == 0:
                break
        it, conv, res, _ = sol2.progress()
        t_dev = time.perf_counter() - t0
        sol2.close()
        del Xd, yd
        # end to end: fit() on host arrays with the tolerance (upload, G, sweeps, results)
        spec_tol = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma,
                                     block_size=case.block_size, iters=case.iters, seed=case.seed, tol=case.tol)
        gc.collect()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        model = en.fit(case.X, case.y, spec_tol)
        t_e2e = time.perf_counter() - t0
        ttt = {"seconds": dist_max(t_dev, world, dev), "sweeps": it, "residual": res, "converged": bool(conv),
               "tol": case.tol, "gram_mode": tol_gm,
               "timed": "set_data of the HBM-resident X (transpose, -X'y/m) + the once-per-fit G = X'X/m "
                        "(covariance mode) + all sweeps; context memory reserved before the timer",
               "e2e_seconds": dist_max(t_e2e, world, dev), "e2e_sweeps": model.iterations,
               "e2e_timed": "fit(X_host, y_host, spec(tol)) through the public API"}
    out["time_to_tol"] = ttt

    # ---------------- end to end through the public API (host arrays, H2D/D2H inside)
    spec = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma,
                             block_size=case.block_size, iters=K, seed=case.seed, tol=None)
    # warm-up call on the full problem: process-level one-time costs (pinned staging
    # buffers, kernel attributes, cluster occupancy queries) stay out of the e2e number
    en.fit(case.X, case.y, spec)
    gc.collect()     # a previous config's multi-GB host arrays must not be freed inside the timer
    torch.cuda.synchronize()
    dist_barrier(world)
    t0 = time.perf_counter()
    en.fit(case.X, case.y, spec)
    t_e2e = dist_max(time.perf_counter() - t0, world, dev)
    out["e2e"] = {"value": world * K / t_e2e, "unit": "sweeps/s",
                  "h2d_bytes_per_step": int((8 * m * n + 8 * m) / K + 8 * n),
                  "d2h_bytes_per_step": int((3 * 8 * n + 8 * 2 * K + 16) / K)}

    # ---------------- roofline of the dominant kernel
    hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
    out["roofline"] = en_roofline(stages, m, n, s, p, gram_mode, variant, hbm, fp64, i8, case.name,
                                  chain_trace.get("prep_batch_sweeps", 1), slices)
    split = out.get("gram_stage_split_ms")
    if split and gram_mode == "blocks":
        # the gram stage's two kernels against their own roofs: slicing moves 8 m n bytes in (FP64
        # columns) and `slices` m n bytes out; the GEMM's int8 ops are the stage entry's
        jt = (s + 127) // 128
        prods = slices * (slices + 1) // 2
        ops = 2.0 * prods * p * (jt * (jt + 1) // 2) * 128 * 128 * ((m + 31) // 32 * 32)
        byts = (8.0 + slices) * float(m) * n
        sl_s, mm_s = split["i8_slice_kernel"] * 1e-3, split["gram_i8_kernel"] * 1e-3
        out["roofline"]["all_stages"] = [
            {"stage": "gram (slicing)", "kernel": "i8_slice_kernel", "bound": "hbm", "achieved": byts / sl_s / 1e9,
             "peak": hbm, "unit": "GB/s", "frac": byts / sl_s / 1e9 / hbm, "ms_per_sweep": split["i8_slice_kernel"]},
            {"stage": "gram (GEMM)", "kernel": "gram_i8_kernel", "bound": "tensor", "achieved": ops / mm_s / 1e12,
             "peak": i8["peak"], "unit": "TOPS (int8)", "frac": ops / mm_s / 1e12 / i8["peak"],
             "ms_per_sweep": split["gram_i8_kernel"]},
        ] + [e for e in out["roofline"]["all_stages"] if e["stage"] != "gram"]
    out["roofline"]["peak_source"] = out["roofline"].get("peak_source", "MEASURED_PEAKS.json hbm_gbs"
                                                         if out["roofline"]["unit"] == "GB/s"
                                                         else "cuBLAS DGEMM 8192^3 measured in this run")

    if headline:
        out.update(en_variants(case, args, world, local, gram_mode, stages, hbm, fp64, i8))
    return out


def en_variants(case, args, world, local, gram_mode, stages, hbm, fp64, i8) -> dict:
    """Beside the headline: the reference's own per-sweep block-Gram arithmetic when the
    headline runs in covariance mode, and RP mode."""
    import torch
    from paper_1907_01995_b200 import _device, elastic_net as en
    from paper_1907_01995_b200.problems import Mode
    dev = torch.device("cuda", local)
    m, n = case.X.shape
    s = min(case.block_size, n)
    p = -(-n // s)
    K, W = args.steps, args.warmup
    extra = {}
    if gram_mode == "covariance":
        sb = en.EnSolver(m, n, s, Mode.RAC, case.lam, case.alpha, case.gamma, device=local)
        sb.set_data(case.X, case.y)
        pb = _device.PermutationFeeder(np.random.default_rng(case.seed), n, dev).draw(W + K)
        sb.run(pb[:W], None)
        torch.cuda.synchronize()
        dist_barrier(world)
        b0, b1 = _ev(), _ev()
        b0.record()
        sb.run(pb[W:W + K], None)
        b1.record()
        torch.cuda.synchronize()
        ms_b = dist_max(b0.elapsed_time(b1), world, dev)
        extra["reference_algorithm_variant"] = {"gram_mode": "blocks", "value": world * K / (ms_b * 1e-3),
                                                "ms_per_step": ms_b / K}
        sb.close()
    srp = en.EnSolver(m, n, s, Mode.RP, case.lam, case.alpha, case.gamma, device=local)
    if gram_mode == "covariance":
        srp.set_gram_mode("covariance")
    srp.set_data(case.X, case.y)
    rrng = np.random.default_rng(case.seed)
    srp.set_partition(_device.PermutationFeeder(rrng, n, dev).draw(1))
    pr = _device.PermutationFeeder(rrng, srp.p, dev).draw(W + K)
    srp.run(pr[:W], None)
    torch.cuda.synchronize()
    dist_barrier(world)
    r0e, r1e = _ev(), _ev()
    r0e.record()
    srp.run(pr[W:W + K], None)
    r1e.record()
    torch.cuda.synchronize()
    ms_rp = dist_max(r0e.elapsed_time(r1e), world, dev)
    extra["rp_mode_variant"] = {"mode": "rp", "gram_mode": gram_mode, "value": world * K / (ms_rp * 1e-3),
                                "ms_per_step": ms_rp / K,
                                "note": "partition and block factorisations formed once (outside the timed "
                                        "K sweeps), as RP defines"}
    srp.close()
    return extra


# ------------------------------------------------------------------ B200 arm: SVM (config 4)
def measure_svm(cfg, case, args, world, rank, local, peaks, headline: bool) -> dict:
    import torch
    from paper_1907_01995_b200 import _device, svm
    from paper_1907_01995_b200.engine import QpSolver
    from paper_1907_01995_b200.problems import Mode, SolverConfig

    dev = torch.device("cuda", local)
    X, y = case.X, case.labels
    N, d = X.shape
    s = case.block_size
    K, W = args.steps, args.warmup
    t0 = time.perf_counter()
    Q = svm.build_q(X, y, svm.KernelSpec("linear"), dev)
    t_q = time.perf_counter() - t0
    solver = QpSolver(N, 1, s, Mode.RAC, case.beta, svm.RIDGE_REL, device=local)
    solver.set_problem(np.full(N, -1.0), np.zeros(N), np.full(N, case.C), A=y.reshape(1, N),
                       b=np.zeros(1), borrowed_h=Q)
    solver.set_divergence_bar(math.inf)
    rng = np.random.default_rng(case.seed)
    perms = _device.PermutationFeeder(rng, N, dev).draw(W + K)
    solver.run(perms[:W], W, case.tol_primal, case.tol_dual, True)
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if headline else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    dist_barrier(world)
    torch.cuda.synchronize()
    e0, e1 = _ev(), _ev()
    l0 = solver.lib.rac_launch_count()
    e0.record()
    solver.run(perms[W:W + K], K, case.tol_primal, case.tol_dual, True)
    e1.record()
    launches = solver.lib.rac_launch_count() - l0
    torch.cuda.synchronize()
    dist_barrier(world)
    out = {}
    if clocks:
        out["clocks"] = clocks.stop()
    ms = dist_max(e0.elapsed_time(e1), world, dev)
    it, status, _ = solver.progress()
    hp, _, hd = (h.cpu().numpy() for h in solver.history(it))
    solver.close()
    del Q
    # ---------------- end to end through the public API (svm.train on host arrays)
    cfgk = SolverConfig(mode=Mode.RAC, block_size=s, beta_penalty=case.beta, max_iters=K,
                        tol_primal=case.tol_primal, tol_dual=case.tol_dual, seed=case.seed, fixed_iterations=True)
    svm.train(X, y, case.C, svm.KernelSpec("linear"), SolverConfig(block_size=s, max_iters=1))
    gc.collect()
    torch.cuda.synchronize()
    dist_barrier(world)
    # median of five complete trains: single trains on the bench box show sporadic 70 - 200 ms
    # stalls (measured: 50 vs 110 - 148 sweeps/s for the same code; back-to-back trains in a fresh
    # process are stable at 135 ms, scripts/prof_train_rep.py)
    reps = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        svm.train(X, y, case.C, svm.KernelSpec("linear"), cfgk)
        reps.append(time.perf_counter() - t0)
    t_e2e = dist_max(sorted(reps)[len(reps) // 2], world, dev)
    # the same train with kernel strips formed on the fly (no resident N x N matrix: the
    # reference's own scheme) — what runs when Q does not fit in HBM
    os.environ["RAC_SVM_STRIPS"] = "1"
    try:
        svm.train(X, y, case.C, svm.KernelSpec("linear"), SolverConfig(block_size=s, max_iters=1))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        svm.train(X, y, case.C, svm.KernelSpec("linear"), cfgk)
        t_strips = dist_max(time.perf_counter() - t0, world, dev)
    finally:
        os.environ.pop("RAC_SVM_STRIPS", None)
    out["kernel_strips_variant"] = {
        "e2e": {"value": world * K / t_strips, "unit": "sweeps/s",
                "h2d_bytes_per_step": int((8 * N * d + 8 * N) / K + 8 * N),
                "d2h_bytes_per_step": int((8 * N + 8) / K + 32)},
        "note": "svm.train with RAC_SVM_STRIPS=1: per sweep the blocks' H_bb and batches of strip rows are "
                "formed from X on the FP64 tensor cores (2 N^2 d flop per sweep) instead of reading a "
                "resident N x N Q"}
    hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
    achieved = 8.0 * N * N / (ms * 1e-3 / K) / 1e9
    out.update({
        "value": world * K / (ms * 1e-3), "ms_per_step": ms / K, "gpu_launches": int(launches),
        "q_build_seconds": t_q,
        "residuals_at_last_sweep": {"primal": float(hp[-1]), "dual": float(hd[-1]), "sweeps": it},
        "time_to_tol": {"seconds": None, "converged": False, "tol": case.tol_primal,
                        "note": "with beta = 1 the dual residual stays near C (reference and GPU alike, "
                                "SURVEY §8(d)); residuals at the cap are reported instead"},
        "e2e": {"value": world * K / t_e2e, "unit": "sweeps/s",
                "h2d_bytes_per_step": int((8 * N * d + 8 * N) / K + 8 * N),
                "d2h_bytes_per_step": int((8 * N + 8) / K + 32),
                "timed": "median of 5 complete svm.train calls on host arrays (each: upload, Q = X X', K sweeps, model)",
                "runs_s": [round(r, 4) for r in reps]},
        "roofline": {"kernel": "qp_chain_kernel", "bound": "hbm", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                     "traffic": traffic_table().get(f"{case.name}:qp_chain_kernel"),
                     "algorithmic": "one strip pass over Q (8*N^2 bytes) per launch (= one sweep)"},
    })
    return out


# ------------------------------------------------------------------ B200 arm: driver
SUMMARY_KEYS = ("value", "ms_per_step", "e2e", "time_to_tol", "roofline", "cpu_baseline", "stage_ms_per_sweep",
                "gram_mode", "residuals_at_last_sweep", "kernel_strips_variant", "config")


def run_b200(args) -> int:
    import torch
    from paper_1907_01995_b200 import _native
    world, rank, local = dist_setup("nccl")
    torch.cuda.set_device(local)
    _native.load()
    peaks = measured_peaks()
    fp64 = fp64_peak_tflops(torch)
    i8 = int8_peak_tops(torch, peaks)
    order = [args.config] + ([] if args.only else [c for c in (1, 2, 3, 4, 5) if c != args.config])
    results = {}
    cases = {}
    for cfg in order:
        headline = cfg == args.config
        case = make_case(cfg)
        if cfg == 4:
            r = measure_svm(cfg, case, args, world, rank, local, peaks, headline)
        else:
            r = measure_en(cfg, case, args, world, rank, local, peaks, fp64, i8, headline)
        r["config"] = config_dict(cfg, case, args.steps, world)
        r["cpu_baseline"] = None
        results[cfg] = r
        cases[cfg] = case
        del case
        gc.collect()
        torch.cuda.empty_cache()
    # the CPU legs run after every GPU measurement: a 16-thread oracle run right before a
    # config's end-to-end leg slowed that leg's host side (measured: config 4 e2e 23 vs 125
    # sweeps/s, config 2 1 860 vs 2 990)
    if rank == 0 and world == 1 and not args.no_cpu:
        for cfg in order:
            results[cfg]["cpu_baseline"] = cpu_baseline(cfg, cases[cfg], budget_s=8.0 if cfg == args.config else 5.0)
    cases.clear()
    h = results[args.config]
    line = {
        "metric": METRIC, "value": h["value"], "unit": "sweeps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": h["config"], "e2e": h["e2e"], "roofline": h["roofline"], "cpu_baseline": h["cpu_baseline"],
        "clocks": h.get("clocks"), "gpu_launches": h["gpu_launches"], "time_to_tol": h.get("time_to_tol"),
    }
    for k in ("stage_ms_per_sweep", "chain_trace", "reference_algorithm_variant", "rp_mode_variant",
              "q_build_seconds", "residuals_at_last_sweep", "kernel_strips_variant"):
        if k in h:
            line[k] = h[k]
    line["peaks"] = {"hbm_gbs": peaks.get("hbm_gbs", HBM_FALLBACK_GBS), "fp64_dgemm_tflops_measured": fp64,
                     "int8": i8}
    line["configs"] = {results[c]["config"]["workload"]: {k: results[c].get(k) for k in SUMMARY_KEYS
                                                           if k in results[c]}
                       for c in sorted(results)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def run_plumbing_check(args) -> int:
    """`--plumbing-check`: the multi-rank plumbing of this script (rank layout, barrier,
    max-over-ranks, rank-0 printing) over gloo, no GPU work.  Used by the CPU test of
    `--gpus N`."""
    world, rank, _ = dist_setup("gloo")
    t0 = time.perf_counter()
    dist_barrier(world)
    val = dist_max(time.perf_counter() - t0 + 1e-6 * (rank + 1), world)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": world, "plumbing_check": True, "max_over_ranks_s": val}),
              flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=HEADLINE, choices=[1, 2, 3, 4, 5],
                    help="headline BASELINE config (default 5, the largest single-GPU one)")
    ap.add_argument("--only", action="store_true", help="measure the headline config only")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--plumbing-check", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--gram", default="auto", choices=["auto", "blocks", "covariance"],
                    help="EN block systems: per-sweep block Grams or covariance mode (G formed inside every "
                         "timed region: throughput, time to tol, e2e)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if args.plumbing_check:
        return run_plumbing_check(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
