"""Print the kernel plan the host compiler picks for c1..c5 (no GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1110_2561_b200 import _native
from paper_1110_2561_b200.workloads import workloads
from paper_1110_2561_b200.enumeration import native_lattice
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))  # noqa: E402
import knobs_env  # noqa: E402
knobs_env.apply()
for k,w in workloads().items():
    t=time.time()
    ok,p=_native.plan(native_lattice(w.spec), w.spec.num_configs)
    print(k, ok, f"{time.time()-t:.2f}s", {f:getattr(p,f) for f in ('l','e_mode','row_words','e_words','plane_words','hist_words','base_words','pair_mode','pair_both','band_rows')}, list(p.pair_degree), list(p.pair_words), f"est={p.est_wavefronts:.3f} per_cfg={p.est_per_config:.3f}", list(p.copy_site))
