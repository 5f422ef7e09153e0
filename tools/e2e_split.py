"""Where the e2e step's wall time goes (c5, one GPU): the C call
(isd_enumerate_thermo) against its own device time, and the Python layer
around it (dos_thermo).

    python tools/e2e_split.py [--reps 30]
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import paper_1110_2561_b200 as isd  # noqa: E402
from paper_1110_2561_b200 import _native  # noqa: E402
from paper_1110_2561_b200.enumeration import native_lattice  # noqa: E402
from paper_1110_2561_b200.workloads import workloads  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c5")
    p.add_argument("--reps", type=int, default=30)
    a = p.parse_args()
    wl = workloads()[a.config]
    spec = wl.spec
    f = np.asarray(wl.fields, dtype=np.float64)
    t = np.asarray(wl.temps, dtype=np.float64)
    lat = native_lattice(spec)
    for _ in range(3):
        isd.dos_thermo(spec, f, t)
    c_wall, c_dev, py_wall, lat_ms = [], [], [], []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        _, _, _, total = _native.enumerate_thermo(
            lat, 0, spec.num_configs, [0], abs(spec.coupling), f, t)
        c_wall.append((time.perf_counter() - t0) * 1e3)
        c_dev.append(total)
        t0 = time.perf_counter()
        isd.dos_thermo(spec, f, t)
        py_wall.append((time.perf_counter() - t0) * 1e3)
        t0 = time.perf_counter()
        native_lattice(spec)
        lat_ms.append((time.perf_counter() - t0) * 1e3)
    med = statistics.median
    print(f"{a.config}: device (root events) {med(c_dev):.4f} ms; "
          f"isd_enumerate_thermo via ctypes {med(c_wall):.4f} ms wall; "
          f"dos_thermo {med(py_wall):.4f} ms wall; native_lattice "
          f"{med(lat_ms):.4f} ms")


if __name__ == "__main__":
    main()
