"""GPU tests of the on-disk plan / cubin cache (csrc/cache.cpp).

A walk of >= 2^33 configurations is autotuned on first use; the winner,
its band cost curve and its NVRTC cubins are written to the cache, so a
new process loads them instead of tuning again (cold start).
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, time
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_1110_2561_b200 as isd
from paper_1110_2561_b200 import _native
from paper_1110_2561_b200.enumeration import native_lattice
from paper_1110_2561_b200.workloads import workloads
_native.set_cache_dirs(sys.argv[2] or None)
isd.full_dos(isd.LatticeSpec(2, 2))
spec = workloads()["c4"].spec
lat = native_lattice(spec)
t0 = time.perf_counter()
table, _ = _native.enumerate_host(lat, 0, 1 << 34)
t1 = time.perf_counter()
_, plan = _native.walk_plan(lat, 0, 1 << 34, 0)
print(json.dumps({"ms": (t1 - t0) * 1e3, "sum": int(table.sum()),
                  "plan": _native.plan_fingerprint(plan),
                  "kernel": _native.kernel_info()}))
"""


def _run(cache):
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, cache],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_second_process_reuses_the_tuned_plan(tmp_path):
    cache = str(tmp_path / "cache")
    first = _run(cache)
    names = os.listdir(cache)
    assert any(n.startswith("plan-") for n in names)
    assert any(n.startswith("cubin-") for n in names)
    second = _run(cache)
    assert first["sum"] == second["sum"] == 1 << 34
    assert first["plan"] == second["plan"]
    assert second["kernel"] == "k1_hoisted_jit"
    # no model search, no autotune, no NVRTC: a small fraction of the first
    assert second["ms"] < 0.25 * first["ms"], (first, second)


@pytest.mark.parametrize("where", ["key", "payload"])
def test_corrupt_cache_entries_are_ignored(tmp_path, where):
    cache = str(tmp_path / "cache")
    good = _run(cache)
    for n in os.listdir(cache):
        path = os.path.join(cache, n)
        with open(path, "r+b") as f:
            # inside the stored key (a miss by key), or the last bytes of the
            # payload (a miss by checksum: never a damaged plan or cubin)
            f.seek(20 if where == "key" else os.path.getsize(path) - 8)
            f.write(b"\xff" * 8)
    again = _run(cache)
    assert again["sum"] == good["sum"] == 1 << 34


def test_no_cache_dir_still_works(tmp_path):
    out = _run("")
    assert out["sum"] == 1 << 34
