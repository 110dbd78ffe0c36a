"""Aggregate PC-sampling stalls per CUDA source line from an ncu report.

    python scripts/ncu_lines.py REPORT.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kre:
    args += ["-k", f"regex:{kre}"]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
per = defaultdict(lambda: defaultdict(float))
src = {}
fname = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = (fname, ln)
    src[key] = r[1].strip()
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k or k in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                per[key][k] += float(v or 0)
            except ValueError:
                pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in per.values()) or 1.0
itot = sum(v.get("Instructions Executed", 0) for v in per.values()) or 1.0
ranked = sorted(per.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]
for key, v in ranked:
    s = v["Warp Stall Sampling (All Samples)"]
    st = sorted(((x, k[6:]) for k, x in v.items() if k.startswith("stall_")), reverse=True)[:3]
    print(f"{s / tot * 100:5.1f}% inst {v.get('Instructions Executed', 0) / itot * 100:4.1f}% {key[0]}:{key[1]:<5d} {src[key][:70]:70s} " +
          " ".join(f"{n}={x / max(s, 1) * 100:.0f}%" for x, n in st))
