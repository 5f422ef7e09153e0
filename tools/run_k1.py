"""Run one BASELINE config's full enumeration a few times (profiling driver).

    python tools/run_k1.py --config c5 --reps 3 [--algo auto|canonical]

Prints device ms per walk and configs/s; exits non-zero on a wrong table
(verify_dos).  Used under ncu: the first launches are warm-up.
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1110_2561_b200 as isd  # noqa: E402
from paper_1110_2561_b200 import _native  # noqa: E402
from paper_1110_2561_b200.enumeration import enumerate_range_timed  # noqa: E402
from paper_1110_2561_b200.workloads import workloads  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))  # noqa: E402
import knobs_env  # noqa: E402
knobs_env.apply()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c5")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--algo", default="auto", choices=["auto", "canonical"])
    p.add_argument("--shards", type=int, default=1,
                   help="time shard --index of make_shards(spec, shards) "
                        "(what one rank of a multi-GPU run walks)")
    p.add_argument("--index", type=int, default=0)
    a = p.parse_args()
    algo = _native.ALGO_AUTO if a.algo == "auto" else _native.ALGO_CANONICAL
    spec = workloads()[a.config].spec
    sh = isd.make_shards(spec, a.shards)[a.index]
    for i in range(a.reps):
        table, ms = enumerate_range_timed(spec, sh.start_index, sh.end_index,
                                          algo=algo)
        if a.shards == 1:
            dos = isd.DoSHistogram(spec, table.view("int64"))
            ok = isd.verify_dos(dos).passed
        else:
            ok = int(table.sum()) == sh.size
        print(f"{a.config} rep {i}: {ms:.3f} ms, "
              f"{sh.size / ms / 1e9:.3f} Tconf/s, verify={ok}",
              flush=True)
        if not ok:
            return 1
    from paper_1110_2561_b200.enumeration import native_lattice
    ok, info = _native.walk_plan(native_lattice(spec), sh.start_index,
                                 sh.end_index)
    print(f"  plan: mode={info.e_mode} sites={list(info.copy_site)} "
          f"A,B,P={info.row_words},{info.e_words},{info.plane_words} "
          f"lane_mask={info.lane_mask:#x} est={info.est_wavefronts:.3f}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
