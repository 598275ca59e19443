"""bench.py's JSON contract on CPU: the reference arm (the unmodified reference package when
baseline/_ref is installed, else the oracle port) prints one well-formed line."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg1",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["unit"] == "ms/layer" and d["value"] > 0
    assert d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    for key in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "scaling", "dtype",
                "config", "data"):
        assert key in d, key


def test_arms_share_one_config_dict():
    """The reference arm's `config` is the GPU arm's (bench.workload_config), so the
    driver's same_config check holds; ms_per_step is the measured wall time of a step."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg1",
                        "--steps", "2", "--warmup", "0"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    args = argparse.Namespace(config="cfg1", parallel="tp")
    d_, f_, L, T, _ = bench.CONFIGS["cfg1"]
    assert d["config"] == bench.workload_config(args, T, L, bench.config_ks("cfg1"), 1)
    assert "extrapolation" in d and d["ms_per_step"] > 0
    ex = d["extrapolation"]
    assert ex["t_dense_block_ms"] + ex["t_predicted_block_ms"] <= d["ms_per_step"] * 1.01
