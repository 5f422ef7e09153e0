"""Stage the reference's own test suite against the drop-in (test infra).

    python tools/stage_reference_suite.py [--src /root/reference/pkg/tests]

Copies the reference package's tests (pkg/tests/*.py) into
`reference_suite/` at the repo root — git-ignored, never committed, and not
under tests/ so the CPU suite does not collect it — where they import
`isingdos`, which resolves to this repo's alias package (isingdos/ ->
paper_1110_2561_b200).  `tests/test_reference_suite.py` (GPU) runs them
with `tests/refsuite_plugin.py`, which marks the documented deviations.
The copy is made in this container (the GPU box has no /root/reference)
and travels with the working tree like the built libraries.
"""

import argparse
import glob
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEST = os.path.join(ROOT, "reference_suite")


def stage(src: str) -> list[str]:
    files = sorted(glob.glob(os.path.join(src, "*.py")))
    if not files:
        raise SystemExit(f"no reference tests under {src}")
    os.makedirs(DEST, exist_ok=True)
    for f in glob.glob(os.path.join(DEST, "*.py")):
        os.remove(f)
    for f in files:
        shutil.copy2(f, DEST)
    return [os.path.basename(f) for f in files]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default="/root/reference/pkg/tests")
    a = ap.parse_args()
    names = stage(a.src)
    print(f"staged {len(names)} files into {DEST}: {' '.join(names)}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
