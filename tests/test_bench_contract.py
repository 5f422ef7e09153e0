"""bench.py keeps the harness contract (CPU: the reference arm; GPU: the
B200 arm's JSON line)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, cwd=ROOT,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "2",
              "--warmup", "1"])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup",
                "ms_per_step", "higher_is_better", "scaling", "cpu_baseline",
                "e2e", "config"):
        assert key in d, key
    assert d["value"] > 0 and d["unit"] == "configs/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_b200_arm_line():
    d = _run(["--config", "c2", "--steps", "3", "--warmup", "3",
              "--extra-configs", "", "--cpu-seconds", "1"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup",
                "ms_per_step", "higher_is_better", "scaling", "vs_baseline",
                "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
                "clocks", "cpu_baseline"):
        assert key in d, key
    assert d["config"]["verify_dos_passed"] is True
    assert d["gpu_launches"] >= 3 * 2
    r = d["roofline"]
    assert r["bound"] == "smem-atomic" and 0 < r["frac"] < 1.2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
