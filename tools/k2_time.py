"""Device time of K2 (compaction + thermodynamics) on a BASELINE grid.

    python tools/k2_time.py [--config c5] [--reps 200]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1110_2561_b200 as isd  # noqa: E402
from paper_1110_2561_b200 import _native  # noqa: E402
from paper_1110_2561_b200.workloads import workloads  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))  # noqa: E402
import knobs_env  # noqa: E402
knobs_env.apply()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c5")
    p.add_argument("--reps", type=int, default=200)
    a = p.parse_args()
    wl = workloads()[a.config]
    spec = wl.spec
    table = isd.full_dos(spec).counts
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(table.reshape(-1)).to(dev)
    f = torch.tensor(list(wl.fields), dtype=torch.float64, device=dev)
    tt = torch.tensor(list(wl.temps), dtype=torch.float64, device=dev)
    out = torch.empty(len(wl.fields) * len(wl.temps) * 7, dtype=torch.float64,
                      device=dev)
    st = torch.cuda.current_stream()
    args = (t.data_ptr(), spec.num_spins, spec.num_bonds,
            float(abs(spec.coupling)), f.data_ptr(), len(wl.fields),
            tt.data_ptr(), len(wl.temps), out.data_ptr(), st.cuda_stream)
    for _ in range(10):
        _native.thermo_device(*args)
    # a CUDA graph of `reps` grids: device time per grid without the
    # per-call host overhead (ctypes + launch ~10 us would dominate)
    cap = torch.cuda.Stream()
    cap.wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cargs = args[:-1] + (cap.cuda_stream,)
    with torch.cuda.graph(g, stream=cap):
        for _ in range(a.reps):
            _native.thermo_device(*cargs)
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / a.reps * 1e3
    host = isd.thermo_grid(isd.DoSHistogram(spec, table), wl.fields, wl.temps)
    same = np.array_equal(out.cpu().numpy().reshape(host.shape), host)
    print(f"{a.config}: K2 {us:.1f} us per grid of "
          f"{len(wl.fields) * len(wl.temps)} points (graph of back-to-back grids), "
          f"identical to thermo_grid: {same}")


if __name__ == "__main__":
    main()
