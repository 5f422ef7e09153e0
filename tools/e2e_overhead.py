"""Host overhead of the one-call pipeline (dos_thermo) on the e2e path.

    python tools/e2e_overhead.py
"""
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


def timeit(fn, n=30):
    fn()
    fn()
    t = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        t.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(t)


def main():
    w = workloads()["c5"]
    f = np.asarray(w.fields, dtype=np.float64)
    t = np.asarray(w.temps, dtype=np.float64)
    small = isd.LatticeSpec(2, 2)
    lat = native_lattice(w.spec)
    print("dos_thermo 2x2 + 702-point grid: %.3f ms" %
          timeit(lambda: isd.dos_thermo(small, f, t)))
    print("dos_thermo 2x2, no grid: %.3f ms" %
          timeit(lambda: isd.dos_thermo(small, [], [1.0])))
    print("full_dos 2x2: %.3f ms" % timeit(lambda: isd.full_dos(small)))
    print("enumerate_host 2x2: %.3f ms" % timeit(
        lambda: _native.enumerate_host(native_lattice(small), 0, 16)))
    dev = []

    def c5():
        _, _, _, ms = _native.enumerate_thermo(lat, 0, w.spec.num_configs, [0],
                                               1.0, f, t)
        dev.append(ms)
    wall = timeit(c5)
    print("enumerate_thermo c5: wall %.3f ms, root events %.3f ms" %
          (wall, statistics.median(dev)))
    print("dos_thermo c5: %.3f ms" % timeit(lambda: isd.dos_thermo(w.spec, f, t)))


if __name__ == "__main__":
    main()
