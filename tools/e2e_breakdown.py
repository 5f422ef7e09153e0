"""Wall-clock breakdown of the e2e step (public API, host buffers) on c5.

    python tools/e2e_breakdown.py [--config c5] [--reps 20]
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1110_2561_b200 as isd  # noqa: E402
from paper_1110_2561_b200.workloads import workloads  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))  # noqa: E402
import knobs_env  # noqa: E402
knobs_env.apply()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c5")
    p.add_argument("--reps", type=int, default=20)
    a = p.parse_args()
    wl = workloads()[a.config]
    shard = isd.make_shards(wl.spec, 1)[0]
    import numpy as np
    fields = np.asarray(wl.fields, dtype=np.float64)  # host input data,
    temps = np.asarray(wl.temps, dtype=np.float64)    # built once (bench.py)
    dos = isd.enumerate_shard(wl.spec, None, shard)
    isd.thermo_grid(dos, fields, temps)
    t_enum, t_thermo, t_dev = [], [], []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        dos = isd.enumerate_shard(wl.spec, None, shard)
        t1 = time.perf_counter()
        isd.thermo_grid(dos, fields, temps)
        t2 = time.perf_counter()
        t_enum.append((t1 - t0) * 1e3)
        t_thermo.append((t2 - t1) * 1e3)
        _, ms = isd.enumeration.enumerate_range_timed(wl.spec, 0,
                                                      wl.spec.num_configs)
        t_dev.append(ms)
    med = statistics.median
    print(f"{a.config}: enumerate_shard {med(t_enum):.3f} ms wall "
          f"(device {med(t_dev):.3f} ms), thermo_grid {med(t_thermo):.3f} ms "
          f"wall for {len(wl.fields) * len(wl.temps)} points")


if __name__ == "__main__":
    main()
