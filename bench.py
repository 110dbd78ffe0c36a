"""Benchmark: RAC-ADMM sweeps/sec (and time to 1e-6) on one B200, vs the CPU reference path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C]

A "step" is one RAC sweep (one pass of the Gauss-Seidel chain over all p
blocks, including that sweep's block assembly, block Grams and factorizations).
The headline workload is BASELINE.json configs[1] (LASSO, D 10000x2000, s=100);
`--config` selects another BASELINE config.  Multi-GPU: the sweep is a
sequential Gauss-Seidel chain, so N>1 runs N independent replicas (one per GPU,
`scaling: weak`) — see DESIGN.md "Multi-GPU".
"""

from __future__ import annotations

import argparse
import glob
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


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
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "gloo" if args.impl == "reference" else "nccl"
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
def en_case(cfg: int):
    from paper_1907_01995_b200 import configs
    return configs.GENERATORS[cfg]()


def en_flops_bytes(m, n, s):
    """Algorithmic work per sweep: Gram m*n*(s+1) flop, D read 8*m*n bytes."""
    return float(m) * n * (s + 1), 8.0 * m * n


def traffic_table() -> dict:
    """DRAM bytes per launch from the committed ncu --set full captures (profiles/*traffic*.json)."""
    out = {}
    for path in sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                              "*traffic*.json"))):
        try:
            with open(path) as f:
                out.update(json.load(f))
        except (OSError, ValueError):
            pass
    return out


INT8_DENSE_TOPS_NOMINAL = 4500.0   # B200 dense INT8 (no measured int8 figure in MEASURED_PEAKS.json)


def block_grams_int8(s: int, p: int, sms: int = 148) -> bool:
    """Mirror of the context's rule (csrc/en.cu rac_en_create): block-mode Grams run on the
    int8 tensor cores when a sweep's 128 x 128 tiles fill the SMs four times."""
    mode = int(os.environ.get("RAC_BG_I8", "1"))
    jt = (s + 127) // 128
    return mode == 2 or (mode == 1 and s >= 128 and p * jt * (jt + 1) // 2 >= 4 * sms)


def covariance_gram_timing(X, dev, reps: int = 3) -> dict:
    """G = X'X/m of the covariance mode, CUDA-event timed (average of `reps` after one
    warm-up) for the int8 digit-slice kernel (method 1: 36 int8 slice products per tile,
    csrc/gram_i8.cu) and the FP64 DMMA tiles (method 0)."""
    import ctypes as C

    import torch
    from paper_1907_01995_b200 import _native
    lib = _native.load()
    m, n = X.shape
    Xc = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev)
    G = torch.empty((n, n), dtype=torch.float64, device=dev)
    out = {}
    for meth, name in ((1, "int8_slices"), (0, "fp64_dmma")):
        call = lambda: _native.check(lib.rac_gram_covariance(C.c_void_p(Xc.data_ptr()), m, m, n,
                                                              C.c_void_p(G.data_ptr()), float(m), meth))
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_ms"] = e0.elapsed_time(e1) / reps
    jt = (n + 127) // 128
    kpad = (m + 31) // 32 * 32
    ops = 2.0 * 36 * (jt * (jt + 1) // 2) * 128 * 128 * kpad      # int8 ops issued (full 128x128 tiles)
    tops = ops / (out["int8_slices_ms"] * 1e-3) / 1e12
    out.update({"int8_tops": tops, "int8_peak_tops": INT8_DENSE_TOPS_NOMINAL,
                "int8_frac": tops / INT8_DENSE_TOPS_NOMINAL,
                "algorithmic": "36 int8 slice products x 2*128*128*K per upper-triangle tile (incl. slicing "
                               "and exponent passes in the time)"})
    del Xc, G
    return out


def en_roofline(stages, m, n, s, p, gram_mode, variant, hbm, fp64, workload, prep_batch=1) -> dict:
    """Roofline entry for the dominant stage of an EN sweep (per-unit figures: SURVEY.md §8(d)).

    `stages` are per-sweep times measured serially; in the pipelined run the
    block systems of `prep_batch` sweeps are prepared by one launch that overlaps
    the chain, so the stage that bounds a sweep is picked on factor / prep_batch."""
    eff = dict(stages)
    eff["factor"] = stages.get("factor", 0.0) / max(1, prep_batch)
    dom = max(eff, key=eff.get)
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
    elif dom == "gram" and block_grams_int8(s, p):
        jt = (s + 127) // 128
        ops = 2.0 * 36 * p * (jt * (jt + 1) // 2) * 128 * 128 * ((m + 31) // 32 * 32)
        achieved = ops / sec / 1e12
        roof = {"kernel": "i8_slice_kernel + gram_i8_kernel (tcgen05 kind::i8)", "bound": "tensor",
                "achieved": achieved, "peak": INT8_DENSE_TOPS_NOMINAL, "unit": "TOPS (int8)",
                "frac": achieved / INT8_DENSE_TOPS_NOMINAL,
                "algorithmic": "36 int8 digit-slice products x 2*128*128*K per upper tile of each of the p "
                               "blocks per sweep (exact FP64 block Grams); peak = B200 dense INT8 (nominal, "
                               "no measured int8 figure)"}
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
    roof["traffic"] = traffic_table().get(f"{workload}:{roof['kernel']}")
    return roof


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


def cpu_en_rate(case, sweeps: int) -> tuple[float, float]:
    """Oracle (numpy restatement of racml fit) sweeps/s over `sweeps` fixed sweeps."""
    from oracle import rac_oracle as ro
    t0 = time.perf_counter()
    ro.en_fit(case.X, case.y, case.lam, case.alpha, case.gamma, case.block_size, sweeps,
              seed=case.seed, tol=None)
    dt = time.perf_counter() - t0
    return sweeps / dt, dt


def cpu_svm_rate(case, sweeps: int) -> tuple[float, float]:
    """Oracle (numpy restatement of racml train) sweeps/s over `sweeps` sweeps (Q formed once, untimed)."""
    from oracle import rac_oracle as ro
    t0 = time.perf_counter()
    ro.svm_train(case.X, case.labels, case.C, "linear", block_size=case.block_size, beta=case.beta,
                 max_iters=sweeps, seed=0)
    dt = time.perf_counter() - t0
    return sweeps / dt, dt


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm on the host cores (oracle port)."""
    case = en_case(args.config)
    if rank != 0:
        return 0
    svm_cfg = args.config == 4
    rate_fn = cpu_svm_rate if svm_cfg else cpu_en_rate
    rate_fn(case, 1)     # warm-up (BLAS threads, page-in)
    total = 0.0
    for _ in range(args.steps):
        _, dt = rate_fn(case, 1)
        total += dt
    rate = args.steps / total
    if svm_cfg:
        N, d = case.X.shape
        cfg = {"workload": case.name, "N": N, "d": d, "block_size": case.block_size}
        sample = f"{args.steps} single-sweep trains of {case.name} (oracle/rac_oracle.svm_train, Q build included)"
    else:
        m, n = case.X.shape
        cfg = {"workload": case.name, "m": m, "n": n, "block_size": case.block_size}
        sample = f"{args.steps} single sweeps of {case.name} (oracle/rac_oracle.en_fit)"
    line = {
        "impl": "reference", "metric": "rac_admm_sweeps_per_sec", "value": rate,
        "unit": "sweeps/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY.md §8(d) seed-0 recipe)",
        "config": cfg,
        "cpu_baseline": {"value": rate, "unit": "sweeps/s", "cores": cpu_threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_b200(args, world, rank, local):
    if args.config == 4:
        return run_b200_svm(args, world, rank, local)
    return run_b200_en(args, world, rank, local)


def run_b200_en(args, world, rank, local):
    import torch
    from paper_1907_01995_b200 import _device, elastic_net as en
    from paper_1907_01995_b200.problems import Mode

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    case = en_case(args.config)
    m, n = case.X.shape
    s = min(case.block_size, n)
    p = -(-n // s)


    # ---------------- device-resident throughput (fixed sweeps, every sweep does full work)
    K, W = args.steps, args.warmup
    gram_mode = args.gram if args.gram != "auto" else en.choose_gram_mode(m, n, s, K)
    solver = en.EnSolver(m, n, s, Mode.RAC, case.lam, case.alpha, case.gamma, device=local)
    if gram_mode == "covariance":
        solver.set_gram_mode("covariance")
    solver.set_data(case.X, case.y)
    rng = np.random.default_rng(case.seed)
    perms = _device.PermutationFeeder(rng, n, dev).draw(W + K)
    torch.cuda.synchronize()
    solver.run(perms[:W], None)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    dist_barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = solver.lib.rac_launch_count()
    e0.record()
    if gram_mode == "covariance":
        solver.set_gram_mode("covariance")   # G = X'X/m is re-formed INSIDE the timed region
    solver.run(perms[W:W + K], None)
    e1.record()
    launches = solver.lib.rac_launch_count() - l0
    torch.cuda.synchronize()
    dist_barrier(world)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    ms = dist_max(ms, world, dev)
    value = world * K / (ms * 1e-3)

    # ---------------- per-stage breakdown (separate sweeps, CUDA events between stages)
    lib = solver.lib
    lib.rac_en_set_timing(solver.h, 1)
    more = _device.PermutationFeeder(rng, n, dev).draw(K)
    solver.run(more, None)
    stage = (np.ctypeslib.ctypes.c_double * 4)()
    nt = np.ctypeslib.ctypes.c_int32()
    lib.rac_en_timing(solver.h, stage, nt)
    stages = {k: float(v) / max(nt.value, 1) for k, v in zip(("assembly", "gram", "factor", "chain"), stage)}
    # chain phase trace (CTA 0 %globaltimer at each phase boundary of one sweep)
    lib.rac_en_set_timing(solver.h, 2)
    solver.run(_device.PermutationFeeder(rng, n, dev).draw(1), None)
    torch.cuda.synchronize()
    ntr = 16 + 16 * p + s
    tbuf = (np.ctypeslib.ctypes.c_int64 * ntr)()
    lib.rac_en_trace(solver.h, tbuf, ntr)
    info = (np.ctypeslib.ctypes.c_int32 * 4)()
    lib.rac_en_info(solver.h, info)
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
    if nl:
        pro = {0: 2, 1: 5, 2: 1, 3: 1}[int(info[0])]   # stamps before the first block
        if info[0] == 3:
            chain_trace.update({"prep_batch_sweeps": int(info[2]), "lookahead_depth": int(info[3])})
        tv = np.array(tbuf[:pro + nl * p], dtype=np.float64) / 1e3   # us
        ph = np.diff(tv[pro - 1:]).reshape(p, nl) if p > 0 else np.zeros((0, nl))
        if info[0] != 3:
            chain_trace.update({"rows_per_chunk": int(info[2]), "chunks_per_cta": int(info[3])})
        chain_trace.update({
                            "first_phase_us": float(tv[pro - 1] - tv[0]),
                            "per_block_us": {k: float(v) for k, v in zip(labels, ph.mean(axis=0))}})
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
    solver.close()
    del perms, more

    # ---------------- time to tolerance (device-resident inputs, host PCG64 stream as in fit)
    ttt = None
    if case.tol is not None:
        sol2 = en.EnSolver(m, n, s, Mode.RAC, case.lam, case.alpha, case.gamma, device=local)
        if args.gram == "covariance" or (args.gram == "auto" and
                                         en.choose_gram_mode(m, n, s, case.iters) == "covariance"):
            sol2.set_gram_mode("covariance")
        sol2.set_data(case.X, case.y)
        rng2 = np.random.default_rng(case.seed)
        feeder = _device.PermutationFeeder(rng2, n, dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # as fit() with a tolerance: batches of 16 sweeps, batch k+1 enqueued before batch
        # k's status is polled; the final progress() reports the converged sweep
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
        t_tol = time.perf_counter() - t0
        ttt = {"seconds": t_tol, "sweeps": it, "residual": res, "converged": bool(conv),
               "tol": case.tol}
        sol2.close()

    # ---------------- end to end through the public API (host arrays, H2D/D2H inside)
    spec = en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma,
                             block_size=case.block_size, iters=K, seed=case.seed, tol=None)
    # warm-up call on the full problem: process-level one-time costs (pinned staging
    # buffers, kernel attributes, cluster occupancy queries) stay out of the e2e number
    en.fit(case.X, case.y, en.ElasticNetSpec(lam=case.lam, alpha=case.alpha, gamma=case.gamma,
                                             block_size=case.block_size, iters=K, seed=case.seed, tol=None))
    torch.cuda.synchronize()
    dist_barrier(world)
    t0 = time.perf_counter()
    en.fit(case.X, case.y, spec)
    t_e2e = time.perf_counter() - t0
    t_e2e = dist_max(t_e2e, world, dev)
    e2e = {"value": world * K / t_e2e, "unit": "sweeps/s",
           "h2d_bytes_per_step": int((8 * m * n + 8 * m) / K + 8 * n),
           "d2h_bytes_per_step": int((3 * 8 * n + 8 * 2 * K + 16) / K)}

    # ---------------- roofline of the dominant kernel
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
    fp64 = fp64_peak_tflops(torch)
    roof = en_roofline(stages, m, n, s, p, gram_mode, chain_trace["variant"], hbm, fp64, case.name,
                       chain_trace.get("prep_batch_sweeps", 1))

    # ---------------- the covariance Gram G = X'X/m (once per fit): int8 digit-slice tensor-core
    # kernel vs the FP64 DMMA tiles, both through rac_gram_covariance on the resident X
    gram_cov = None
    if gram_mode == "covariance":
        gram_cov = covariance_gram_timing(case.X, dev)

    # ---------------- the reference's own algorithm (per-sweep block Grams from X), reported
    # beside the covariance-mode headline (the G-reuse variant's algorithmic
    # work differs, so its roofline is not comparable)
    alt = None
    if gram_mode == "covariance":
        sb = en.EnSolver(m, n, s, Mode.RAC, case.lam, case.alpha, case.gamma, device=local)
        sb.set_data(case.X, case.y)
        pb = _device.PermutationFeeder(np.random.default_rng(case.seed), n, dev).draw(W + K)
        sb.run(pb[:W], None)
        torch.cuda.synchronize()
        dist_barrier(world)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record()
        sb.run(pb[W:W + K], None)
        b1.record()
        torch.cuda.synchronize()
        ms_b = dist_max(b0.elapsed_time(b1), world, dev)
        sb.lib.rac_en_set_timing(sb.h, 1)
        sb.run(_device.PermutationFeeder(rng, n, dev).draw(K), None)
        stb = (np.ctypeslib.ctypes.c_double * 4)()
        ntb = np.ctypeslib.ctypes.c_int32()
        sb.lib.rac_en_timing(sb.h, stb, ntb)
        stages_b = {k: float(v) / max(ntb.value, 1) for k, v in zip(("assembly", "gram", "factor", "chain"), stb)}
        infb = (np.ctypeslib.ctypes.c_int32 * 4)()
        sb.lib.rac_en_info(sb.h, infb)
        var_b = {0: "streaming", 1: "resident-cluster"}.get(int(infb[0]), "streaming")
        alt = {"gram_mode": "blocks", "value": world * K / (ms_b * 1e-3), "ms_per_step": ms_b / K,
               "stage_ms_per_sweep": stages_b, "chain_variant": var_b,
               "roofline": en_roofline(stages_b, m, n, s, p, "blocks", var_b, hbm, fp64, case.name)}
        sb.close()
        del pb

    # ---------------- RP mode: fixed partition, block systems formed
    # once at set_partition, per-sweep block ORDER permutation; the chain is the whole sweep
    rp = None
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
    r0e, r1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0e.record()
    srp.run(pr[W:W + K], None)
    r1e.record()
    torch.cuda.synchronize()
    ms_rp = dist_max(r0e.elapsed_time(r1e), world, dev)
    rp = {"mode": "rp", "gram_mode": gram_mode, "value": world * K / (ms_rp * 1e-3), "ms_per_step": ms_rp / K,
          "note": "partition and block factorisations formed once (outside the timed K sweeps), as RP defines"}
    srp.close()
    del pr

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r1, dt1 = cpu_en_rate(case, 1)
        sweeps = int(max(1, min(60, 15.0 / max(dt1, 1e-3))))
        rate, dt = cpu_en_rate(case, sweeps)
        cpu = {"value": rate, "unit": "sweeps/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"{sweeps} sweeps of {case.name} via oracle/rac_oracle.en_fit ({dt:.1f} s)"}

    line = {
        "metric": "rac_admm_sweeps_per_sec", "value": value, "unit": "sweeps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY.md §8(d) seed-0 recipe)",
        "config": {"workload": case.name, "m": m, "n": n, "block_size": s, "blocks": p,
                   "mode": "rac", "gram_mode": gram_mode,
                   "l2": "inputs larger than L2 (D = %.0f MB)" % (8 * m * n / 1e6)
                   if 8 * m * n > 126e6 else "D fits in L2 (no flush)",
                   "parallelism": f"replicas x{world}"},
        "stage_ms_per_sweep": stages,
        "chain_trace": chain_trace,
        "time_to_tol": ttt,
        "e2e": e2e,
        "roofline": roof,
        "reference_algorithm_variant": alt,
        "rp_mode_variant": rp,
        "covariance_gram": gram_cov,
        "fp64_dgemm_tflops_measured": fp64,
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": int(launches),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_b200_svm(args, world, rank, local):
    """Config 4: linear-SVM dual, N=20000, s=100, dense Q resident in HBM (3.2 GB)."""
    import torch
    from paper_1907_01995_b200 import _device, svm
    from paper_1907_01995_b200.engine import QpSolver
    from paper_1907_01995_b200.problems import Mode, SolverConfig

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_1907_01995_b200 import configs
    case = configs.config4()
    X, y = case.X, case.labels
    N, d = X.shape
    s = case.block_size
    p = -(-N // s)
    t0 = time.perf_counter()
    Q = svm.build_q(X, y, svm.KernelSpec("linear"), dev)
    t_q = time.perf_counter() - t0
    solver = QpSolver(N, 1, s, Mode.RAC, case.beta, svm.RIDGE_REL, device=local)
    solver.set_problem(np.full(N, -1.0), np.zeros(N), np.full(N, case.C), A=y.reshape(1, N),
                       b=np.zeros(1), borrowed_h=Q)
    solver.set_divergence_bar(math.inf)
    rng = np.random.default_rng(case.seed)
    K, W = args.steps, args.warmup
    perms = _device.PermutationFeeder(rng, N, dev).draw(W + K)
    solver.run(perms[:W], W, case.tol_primal, case.tol_dual, True)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    dist_barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = solver.lib.rac_launch_count()
    e0.record()
    solver.run(perms[W:W + K], K, case.tol_primal, case.tol_dual, True)
    e1.record()
    launches = solver.lib.rac_launch_count() - l0
    torch.cuda.synchronize()
    dist_barrier(world)
    clk = clocks.stop()
    ms = dist_max(e0.elapsed_time(e1), world, dev)
    value = world * K / (ms * 1e-3)
    it, status, _ = solver.progress()
    hp, _, hd = (h.cpu().numpy() for h in solver.history(it))
    solver.close()
    # ---------------- end to end through the public API (svm.train on host arrays)
    cfg = SolverConfig(mode=Mode.RAC, block_size=s, beta_penalty=case.beta, max_iters=K,
                       tol_primal=case.tol_primal, tol_dual=case.tol_dual, seed=0, fixed_iterations=True)
    svm.train(X, y, case.C, svm.KernelSpec("linear"), SolverConfig(block_size=s, max_iters=1))
    torch.cuda.synchronize()
    dist_barrier(world)
    t0 = time.perf_counter()
    svm.train(X, y, case.C, svm.KernelSpec("linear"), cfg)
    t_e2e = dist_max(time.perf_counter() - t0, world, dev)
    e2e = {"value": world * K / t_e2e, "unit": "sweeps/s",
           "h2d_bytes_per_step": int((8 * N * d + 8 * N) / K + 8 * N),
           "d2h_bytes_per_step": int((8 * N + 8) / K + 32)}
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
    strip_bytes = 8.0 * N * N
    achieved = strip_bytes / (ms * 1e-3 / K) / 1e9
    roof = {"kernel": "qp_chain_kernel", "bound": "hbm", "achieved": achieved, "peak": hbm,
            "unit": "GB/s", "frac": achieved / hbm,
            "traffic": traffic_table().get(f"{case.name}:qp_chain_kernel"),
            "algorithmic": "one strip pass over Q (8*N^2 bytes) per launch (= one sweep)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import rac_oracle as ro
        t0 = time.perf_counter()
        ro.svm_train(X, y, case.C, "linear", block_size=s, beta=case.beta, max_iters=1, seed=0)
        dt = time.perf_counter() - t0
        cpu = {"value": 1.0 / dt, "unit": "sweeps/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"1 sweep of {case.name} via oracle/rac_oracle.svm_train ({dt:.1f} s)"}
    line = {
        "metric": "rac_admm_sweeps_per_sec", "value": value, "unit": "sweeps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY.md §8(d) seed-0 recipe)",
        "config": {"workload": case.name, "N": N, "d": d, "block_size": s, "blocks": p, "mode": "rac",
                   "l2": "inputs larger than L2 (Q = %.1f GB)" % (8 * N * N / 1e9),
                   "parallelism": f"replicas x{world}"},
        "q_build_seconds": t_q,
        "residuals_at_last_sweep": {"primal": float(hp[-1]), "dual": float(hd[-1]), "sweeps": it},
        "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": int(launches),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--gram", default="auto", choices=["auto", "blocks", "covariance"],
                    help="EN block systems: per-sweep block Grams or covariance mode (G formed in the timed region)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        rc = run_reference(args, world, rank)
    else:
        rc = run_b200(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
