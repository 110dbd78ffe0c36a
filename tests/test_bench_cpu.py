"""bench.py's contract on CPU: the reference arm (oracle port on the host cores) prints one
JSON line with the driver's keys, and the argument surface the driver uses parses."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1"])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["metric"] == "rac_admm_sweeps_per_sec" and d["unit"] == "sweeps/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "ridge_2000x500_s50"


def test_help_lists_driver_flags():
    out = subprocess.run([sys.executable, "bench.py", "--help"], cwd=ROOT, capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl"):
        assert flag in out.stdout


def test_reference_config_matches_b200_arm_config():
    """Both arms print the same `config` object for the same workload (the driver pairs them)."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_1907_01995_b200 import configs
    d = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1"])
    assert d["config"] == bench.config_dict(1, configs.config1(), 2, 1)
    assert d["config"]["gram_mode"] in ("blocks", "covariance")


def test_default_headline_is_largest_config():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.HEADLINE == 5


def test_gpus_n_launches_n_ranks():
    """`--gpus 2` without torchrun re-launches itself as two ranks (gloo plumbing check)."""
    d = _run(["--gpus", "2", "--plumbing-check"], timeout=300)
    assert d["n_gpus"] == 2 and d["plumbing_check"] is True
