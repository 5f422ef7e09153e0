import sys; sys.path.insert(0, "/root/repo")
import paper_1110_2561_b200 as isd
from paper_1110_2561_b200 import _native
from paper_1110_2561_b200.enumeration import native_lattice
from paper_1110_2561_b200.workloads import workloads
_native.set_knob("ISD_LOOP_BITS", 5)
spec = workloads()["c5"].spec; lat = native_lattice(spec)
shards = isd.make_shards(spec, 8)
for order in ([2], [0,1,2,3]):
    for i in order:
        sh = shards[i]
        t = [_native.enumerate_host(lat, sh.start_index, sh.end_index)[1] for _ in range(3)]
        ok, p = _native.walk_plan(lat, sh.start_index, sh.end_index, 0)
        print(i, [round(x,4) for x in t], _native.kernel_info(), "k", p.k, "l", p.l, "band", p.band_rows, "pair", p.pair_mode, hex(p.lane_mask), [hex(v) for v in p.lane_vec], round(p.est_wavefronts,4), "A", p.row_words, list(p.pair_words), _native.plan_fingerprint(p), flush=True)
