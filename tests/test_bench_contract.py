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
