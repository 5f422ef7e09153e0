"""The reference's own test suite, run against the drop-in on the GPU.

tools/stage_reference_suite.py copies /root/reference/pkg/tests (168 tests)
into reference_suite/ (git-ignored test infrastructure; the GPU box has no
/root/reference).  There they `import isingdos`, which resolves to the
alias package isingdos/ -> paper_1110_2561_b200, so every reference test
exercises this engine through the reference's public API, unchanged.  The
documented deviations are in tests/refsuite_plugin.py.
"""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "reference_suite")


@pytest.mark.gpu
def test_reference_suite_passes_on_the_drop_in():
    if not os.path.exists(os.path.join(SUITE, "conftest.py")):
        pytest.skip("reference suite not staged "
                    "(python tools/stage_reference_suite.py)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(
        [ROOT, os.path.join(ROOT, "tests"), env.get("PYTHONPATH", "")])
    r = subprocess.run(
        [sys.executable, "-m", "pytest", SUITE, "-q", "-p", "refsuite_plugin",
         "-p", "no:cacheprovider", "-rxX"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail + r.stderr[-2000:]
    summary = r.stdout.strip().splitlines()[-1]
    passed = int(re.search(r"(\d+) passed", summary).group(1))
    xfailed = re.search(r"(\d+) xfailed", summary)
    # every reference test ran: only the documented deviations may xfail
    assert passed + (int(xfailed.group(1)) if xfailed else 0) >= 168, summary
    assert not re.search(r"\d+ (failed|error)", summary), summary
