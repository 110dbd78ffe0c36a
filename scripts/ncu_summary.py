"""Summarise Nsight Compute captures for profiles/.

    python scripts/ncu_summary.py REPORT.ncu-rep [...]          -> markdown on stdout
    python scripts/ncu_summary.py --launches LAUNCHES.csv       -> per-kernel launch table
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA inst % of peak (active cycles)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return [r for r in csv.reader(io.StringIO(out))]


def report(path):
    rows = ncu_csv(["-i", path, "--page", "raw", "--csv"])
    if len(rows) < 3:
        print(f"(no kernels in {path})")
        return
    h, units = rows[0], rows[1]
    print(f"### `{path.split('/')[-1]}`\n")
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"**{d.get('Kernel Name', '?')[:100]}**\n")
        print("| metric | value |\n|---|---|")
        for k, label in METRICS:
            if k in d and d[k] not in ("", "n/a"):
                print(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
        stalls = []
        for k in h:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(d[k]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = sorted(stalls, reverse=True)[:6]
        print("\nTop warp-stall reasons (PC sampling): " +
              ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in top) + "\n")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = d["Kernel Name"].split("(")[0]
        try:
            v = float(d["Metric Value"])
        except ValueError:
            continue
        agg[k][0] += 1
        agg[k][1] += v
    ours = {k: v for k, v in agg.items() if "cutlass" not in k and "at::" not in k}
    tot = sum(v[1] for v in ours.values()) or 1.0
    print("| kernel | launches | total us | avg us | share of rac kernels |\n|---|---|---|---|---|")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = f"{v / tot * 100:.1f}%" if k in ours else "(not ours)"
        print(f"| `{k[:70]}` | {n} | {v / 1e3:.1f} | {v / n / 1e3:.2f} | {share} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        for p in sys.argv[2:]:
            launches(p)
    else:
        for p in sys.argv[1:]:
            report(p)
