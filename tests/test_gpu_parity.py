"""GPU parity: the B200 engine vs the reference's goldens and the oracle.

Every test here calls the native engine through the C ABI (ctypes) on
cuda:0.  Integer tables must be bit-exact; thermodynamics within 1e-12
relative (absolute 1e-12 where the reference value is structurally ~0,
e.g. <M> at h = 0), as BASELINE.json's north_star states.
"""

import math
import os
import random
import zlib

import numpy as np
import pytest

import paper_1110_2561_b200 as isd
from paper_1110_2561_b200 import _native
from paper_1110_2561_b200.enumeration import enumerate_range_timed
from paper_1110_2561_b200.workloads import workloads
from golden_io import csv_goldens, load_json, read_csv_table, read_json_table
from oracle import port

pytestmark = pytest.mark.gpu

RTOL = 1e-12
ATOL = 1e-12


def full(spec, algo=_native.ALGO_AUTO):
    table, _ = enumerate_range_timed(spec, 0, spec.num_configs, algo=algo)
    return table.view(np.int64)


def spec_from_csv(name):
    rows, cols, depth, j, table = read_csv_table(name)
    return isd.LatticeSpec(rows, cols, depth, j), table


# -- reference goldens (reference package output, tests/golden/*.csv) ------

@pytest.mark.parametrize("name", csv_goldens())
@pytest.mark.parametrize("algo", [_native.ALGO_AUTO, _native.ALGO_CANONICAL])
def test_reference_golden_tables(name, algo):
    spec, want = spec_from_csv(name)
    got = full(spec, algo)
    assert np.array_equal(got, want), name


@pytest.mark.parametrize("name", [n for n in csv_goldens()
                                  if "x1_" in n or "x2_" in n])
@pytest.mark.parametrize("loop_bits", [1, 4, 7])
def test_reference_goldens_with_forced_loop_width(name, loop_bits, monkeypatch):
    spec, want = spec_from_csv(name)
    if spec.num_spins < 7 + loop_bits + 1:
        pytest.skip("too small for this loop width")
    _native.set_knob("ISD_LOOP_BITS", str(loop_bits))
    got = full(spec, _native.ALGO_HOISTED)
    assert np.array_equal(got, want)


def test_4x4_public_api_equals_80_cell_golden():
    spec, want = spec_from_csv("dos_4x4x1_J1.csv")
    dos = isd.enumerate_shard(spec, isd.build_tables(4),
                              isd.make_shards(spec, 1)[0])
    assert np.array_equal(dos.counts, want)
    assert len(dos.cells()) == 80
    assert dos.total() == 65536
    assert isd.verify_dos(dos).passed


def test_odd_shards_of_5x5_match_reference_slices():
    spec = isd.LatticeSpec(5, 5)
    ref = isd.DoSHistogram(spec)
    for rec in load_json("shards_5x5.json"):
        sh = isd.Shard(rec["shard_id"], rec["num_shards"], rec["start"],
                       rec["end"])
        got = isd.enumerate_shard(spec, None, sh)
        want = isd.DoSHistogram(spec)
        for c, m, e in rec["cells"]:
            want.counts[want.m_index(m), want.e_index(e)] = c
        assert got == want, (rec["num_shards"], rec["shard_id"])


def test_unaligned_tall_column_slice():
    rec = load_json("slice_17x2_123456_4096.json")
    spec = isd.LatticeSpec(17, 2)
    got = isd.enumerate_shard(spec, None,
                              isd.Shard(0, 1, rec["start"], rec["end"]))
    assert got.total() == 4096
    assert got.cells() == [tuple(c) for c in rec["cells"]]


def test_empty_and_invalid_ranges():
    spec = isd.LatticeSpec(2, 2)
    empty = isd.enumerate_shard(spec, None, isd.Shard(0, 1, 5, 5))
    assert empty.total() == 0 and not empty.counts.any()
    with pytest.raises(ValueError):
        isd.enumerate_shard(spec, None, isd.Shard(0, 1, 0, 17))
    with pytest.raises(ValueError):
        isd.enumerate_shard(spec, None, isd.Shard(0, 1, 3, 2))


# -- random ranges vs the oracle port (any lattice, incl. free / +-J) -------

RANGE_SPECS = [
    dict(rows=5, cols=5), dict(rows=3, cols=3, depth=4),
    dict(rows=6, cols=6, boundary="free"), dict(rows=6, cols=6, seed=1234),
    dict(rows=4, cols=4, depth=2, coupling=-1), dict(rows=17, cols=2),
    dict(rows=2, cols=2, depth=9), dict(rows=5, cols=7, seed=3),
    dict(rows=4, cols=10), dict(rows=20, cols=2, seed=9),
]


def _spec(kw):
    kw = dict(kw)
    seed = kw.pop("seed", None)
    spec = isd.LatticeSpec(**kw)
    if seed is not None:
        spec = isd.LatticeSpec(**kw, bond_signs=isd.random_bond_signs(spec, seed))
    return spec


def _port(spec):
    return port.Lattice(spec.rows, spec.cols, spec.depth, spec.coupling,
                        spec.periodic,
                        list(spec.bond_signs) if spec.bond_signs else None)


@pytest.mark.parametrize("kw", RANGE_SPECS)
def test_random_ranges_bit_exact(kw):
    spec = _spec(kw)
    lat = _port(spec)
    rng = random.Random(zlib.crc32(repr(sorted(kw.items())).encode()))
    total = spec.num_configs
    for trial in range(6):
        size = rng.choice([1, 31, 4095, 4097, 1 << 16, (1 << 20) + 12345])
        a = rng.randrange(0, total - size)
        if trial == 0:
            a = total - size  # tail of the space
        b = a + size
        table, _ = enumerate_range_timed(spec, a, b)
        want = port.enumerate_range(lat, a, b)
        assert np.array_equal(table.view(np.int64), want), (a, b)


# -- the five BASELINE lattices at full size ---------------------------------

def _golden_c(name):
    if name == "c5" and os.path.exists(os.path.join(
            os.path.dirname(__file__), "golden", "dos_3x3x4_J1.csv")):
        return read_csv_table("dos_3x3x4_J1.csv")[4]
    fname = {"c1": "c1_4x4_free.json", "c3": "c3_6x6_free.json",
             "c4": "c4_6x6_pmJ_seed1234.json",
             "c5": "cx_3x3x4_periodic.json"}.get(name)
    if name == "c2":
        return read_csv_table("dos_5x5x1_J1.csv")[4]
    path = os.path.join(os.path.dirname(__file__), "golden", fname)
    if not os.path.exists(path):
        pytest.skip(f"golden {fname} not generated yet")
    return read_json_table(fname)[1]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_baseline_lattice_full_walk(name):
    spec = workloads()[name].spec
    got = full(spec)
    assert np.array_equal(got, _golden_c(name))
    dos = isd.DoSHistogram(spec, got)
    assert isd.verify_dos(dos).passed
    if name in ("c1", "c3", "c4"):  # bipartite: g(E) = g(-E) marginal
        e_marg = got.sum(axis=0)
        assert np.array_equal(e_marg, e_marg[::-1])


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("pair", ["0", "1", "2", "3"])
def test_paired_and_unpaired_copies(name, pair, monkeypatch):
    # ISD_PAIR forces the pairing mode: 0 = every copy its own RED, 1 = copy
    # bit 6 paired (2 configurations per RED), 2 = bits 6 and 5 (4 per RED),
    # 3 = bits 4-6 as a cluster of three like sites (8 per RED, multiset
    # planes); every mode must give the golden table (the autotuner then
    # times only layouts of that mode)
    _native.set_knob("ISD_PAIR", pair)
    spec = workloads()[name].spec
    _, info = _native.plan(__import__(
        "paper_1110_2561_b200.enumeration",
        fromlist=["native_lattice"]).native_lattice(spec), spec.num_configs)
    if pair == "2" and info.pair_mode != 2:
        pytest.skip("mode-2 histogram does not fit shared memory")
    if pair == "3" and info.pair_mode != 3:
        pytest.skip("no cluster of three like sites / table does not fit")
    assert info.pair_mode == int(pair)
    assert np.array_equal(full(spec), _golden_c(name))


@pytest.mark.parametrize("name", ["c1", "c3", "c5"])
@pytest.mark.parametrize("variant", ["even", "low"])
def test_copy_site_variants(name, variant, monkeypatch):
    # both copy-site choices (even-degree sites with parity planes, lowest
    # sites) must give the same table; c3/c1 are the free-boundary lattices
    # where the parity planes carry odd-degree sites
    _native.set_knob("ISD_COPY_VARIANT", variant)
    spec = workloads()[name].spec
    lat = __import__("paper_1110_2561_b200.enumeration",
                     fromlist=["native_lattice"]).native_lattice(spec)
    usable, info = _native.plan(lat, spec.num_configs)
    if not usable:
        pytest.skip("variant not available")
    got = full(spec, _native.ALGO_HOISTED)
    assert np.array_equal(got, _golden_c(name))


def test_6x6_periodic_matches_reference_walk():
    path = os.path.join(os.path.dirname(__file__), "golden",
                        "dos_6x6x1_J1.csv")
    if not os.path.exists(path):
        pytest.skip("reference 6x6 golden not generated")
    spec, want = spec_from_csv("dos_6x6x1_J1.csv")
    assert np.array_equal(full(spec), want)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_jit_and_aot_kernels_agree(name, monkeypatch):
    spec = workloads()[name].spec
    jit = full(spec)
    assert _native.kernel_info() == "k1_hoisted_jit"
    _native.set_knob("ISD_JIT", "0")
    aot = full(spec)
    assert _native.kernel_info() == "k1_hoisted_aot"
    assert np.array_equal(jit, aot)
    assert np.array_equal(jit, _golden_c(name))


def test_n36_canonical_equals_hoisted():
    spec = workloads()["c4"].spec
    a = full(spec, _native.ALGO_CANONICAL)
    b = full(spec, _native.ALGO_HOISTED)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_flip_symmetry_half_walk_equals_full_walk(name):
    spec = workloads()[name].spec
    whole = full(spec)
    half, _ = enumerate_range_timed(
        spec, 0, spec.num_configs,
        algo=_native.ALGO_AUTO | _native.FLAG_FLIP_SYMMETRY)
    assert np.array_equal(half.view(np.int64), whole)
    dos = isd.full_dos(spec, workers=3, flip_symmetry=True)
    assert np.array_equal(dos.counts, whole)


def test_flip_symmetry_rejects_partial_ranges():
    spec = isd.LatticeSpec(4, 4)
    with pytest.raises(ValueError, match="full range"):
        enumerate_range_timed(spec, 0, 100,
                              algo=_native.FLAG_FLIP_SYMMETRY)


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_shard_count_invisible_at_n36(shards):
    spec = workloads()["c5"].spec
    whole = full(spec)
    dos, wall, per = isd.full_dos_timed(spec, workers=shards)
    assert np.array_equal(dos.counts, whole)
    assert len(per) == shards and all(p > 0 for p in per) and wall > 0


# -- thermodynamics ---------------------------------------------------------

def _close(got, want, absolute=False):
    if absolute:
        return abs(got - want) <= ATOL
    return abs(got - want) <= RTOL * max(abs(want), 1e-300) or \
        abs(got - want) <= ATOL * 1e-3


FIELDS = ["log_z", "free_energy", "internal_energy", "specific_heat",
          "mean_magnetization", "susceptibility"]


def test_thermo_matches_reference_partition_point():
    cases = load_json("thermo_reference.json")
    for case in cases:
        spec, table = spec_from_csv(case["dos"])
        dos = isd.DoSHistogram(spec, table)
        by_field = {}
        for p in case["points"]:
            by_field.setdefault(float(p[0]), []).append(p)
        for h, pts in by_field.items():
            temps = [float(p[1]) for p in pts]
            got = isd.thermo_sweep(dos, h, temps)
            for g, p in zip(got, pts):
                for i, name in enumerate(FIELDS):
                    want = float(p[2 + i])
                    val = getattr(g, name)
                    structural_zero = name == "mean_magnetization" and h == 0
                    assert _close(val, want, structural_zero), (
                        case["dos"], h, g.temperature, name, val, want)


def test_sweep_first_point_equals_partition_point_exactly():
    spec, table = spec_from_csv("dos_4x4x1_J1.csv")
    dos = isd.DoSHistogram(spec, table)
    temps = [0.5 + 0.05 * i for i in range(91)]
    sweep = isd.thermo_sweep(dos, 0.1, temps)
    assert sweep[0] == isd.partition_point(dos, 0.1, temps[0])
    assert sweep[57] == isd.partition_point(dos, 0.1, temps[57])


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_thermo_grid_vs_oracle_on_baseline_grids(name):
    wl = workloads()[name]
    spec = wl.spec
    table = _golden_c(name)
    dos = isd.DoSHistogram(spec, table)
    out = isd.thermo_grid(dos, wl.fields, wl.temps)
    for fi, h in enumerate(wl.fields):
        for ti, t in enumerate(wl.temps):
            want = port.partition_point(table, spec.num_spins, spec.num_bonds,
                                        abs(spec.coupling), h, t)
            for k, w in enumerate(want):
                structural_zero = k == 4 and h == 0
                assert _close(out[fi, ti, k], w, structural_zero), (
                    name, h, t, k, out[fi, ti, k], w)


def test_thermo_validation():
    spec, table = spec_from_csv("dos_2x2x1_J1.csv")
    dos = isd.DoSHistogram(spec, table)
    with pytest.raises(ValueError, match="temperature"):
        isd.partition_point(dos, 0.0, 0.0)
    with pytest.raises(ValueError, match="strictly increasing"):
        isd.thermo_sweep(dos, 0.0, [1.0, 1.0])
    with pytest.raises(ValueError, match="nonempty"):
        isd.thermo_sweep(dos, 0.0, [])
    half = isd.DoSHistogram(spec, table // 2)
    with pytest.raises(ValueError, match="complete"):
        isd.partition_point(half, 0.0, 1.0)


def test_2x2_closed_form_log_z():
    # Z = 2 e^{8/T} + 12 + 2 e^{-8/T} for the periodic 2x2 (test_thermo.py:14-21)
    spec, table = spec_from_csv("dos_2x2x1_J1.csv")
    dos = isd.DoSHistogram(spec, table)
    for t in (0.5, 1.0, 2.0, 10.0):
        z = 2 * math.exp(8 / t) + 12 + 2 * math.exp(-8 / t)
        assert abs(isd.partition_point(dos, 0.0, t).log_z - math.log(z)) \
            <= 1e-12 * math.log(z)


def test_launch_counter_moves():
    before = _native.launch_count()
    full(isd.LatticeSpec(5, 5))
    assert _native.launch_count() > before


def test_bounds_checked_build_runs_clean():
    # the -DISD_DEBUG_BOUNDS library traps on any shared-histogram address
    # outside the warp's histogram (compute-sanitizer is closed on the pool)
    import subprocess
    import sys
    from paper_1110_2561_b200._build import LIB_DEBUG
    if not os.path.exists(LIB_DEBUG):
        pytest.skip("debug library not built")
    env = dict(os.environ, ISD_LIBRARY=LIB_DEBUG)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import runpy; runpy.run_path(%r)\n"
        "from paper_1110_2561_b200.workloads import workloads\n"
        "from paper_1110_2561_b200.enumeration import enumerate_range_timed\n"
        "import paper_1110_2561_b200 as isd\n"
        "from paper_1110_2561_b200 import _native\n"
        "for pm in ('0', '1', '2'):\n"
        "    _native.set_knob('ISD_PAIR', pm)\n"
        "    for n in ('c3', 'c4', 'c5'):\n"
        "        s = workloads()[n].spec\n"
        "        t, _ = enumerate_range_timed(s, 0, 1 << 33)\n"
        "        assert int(t.sum()) == 1 << 33\n"
        "print('bounds ok')\n"
    ) % (root, os.path.join(root, "tools", "sanitize_case.py"))
    r = subprocess.run([sys.executable, "-c", code], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "bounds ok" in r.stdout


# -- maximum size (N = 40, the reference's cap) : size-independent checks ---

N40 = [
    dict(rows=5, cols=8), dict(rows=4, cols=10, boundary="free"),
    dict(rows=2, cols=4, depth=5), dict(rows=5, cols=8, seed=40),
    dict(rows=20, cols=2, coupling=-1),
    # length-2 periodic axes: double bonds through the JIT kernel
    dict(rows=2, cols=20), dict(rows=2, cols=2, depth=10, seed=3),
]


def _bipartite(spec):
    dims = (spec.rows, spec.cols, spec.depth)
    if not spec.periodic:
        return True
    return all(d % 2 == 0 for d in dims if d > 1)


@pytest.mark.parametrize("kw", N40)
def test_n40_full_walk_invariants(kw):
    spec = _spec(kw)
    assert spec.num_spins == 40
    t = full(spec)
    dos = isd.DoSHistogram(spec, t)
    rep = isd.verify_dos(dos)
    assert rep.passed, str(rep)          # 2^40 total, C(40,k) rows, M flip
    if _bipartite(spec):
        e = t.sum(axis=0)
        assert np.array_equal(e, e[::-1])
    # a slice against the oracle port, and shard-count invisibility
    lat = _port(spec)
    a = (1 << 39) + 987654321
    part, _ = enumerate_range_timed(spec, a, a + (1 << 20) + 7)
    assert np.array_equal(part.view(np.int64),
                          port.enumerate_range(lat, a, a + (1 << 20) + 7))
    three = sum(enumerate_range_timed(spec, s.start_index, s.end_index)[0]
                for s in isd.make_shards(spec, 3))
    assert np.array_equal(three.view(np.int64), t)


def test_n40_canonical_equals_hoisted():
    spec = _spec(dict(rows=5, cols=8, seed=7))
    assert np.array_equal(full(spec, _native.ALGO_CANONICAL), full(spec))


@pytest.mark.parametrize("kw", [dict(rows=2, cols=17), dict(rows=2, cols=2,
                                                           depth=9, seed=5)])
def test_double_bond_lattices_jit_vs_aot(kw, monkeypatch):
    spec = _spec(kw)
    jit = full(spec)
    assert _native.kernel_info() == "k1_hoisted_jit"
    _native.set_knob("ISD_JIT", "0")
    assert np.array_equal(full(spec), jit)
    assert isd.verify_dos(isd.DoSHistogram(spec, jit)).passed


def test_thermo_call_overhead_stays_small():
    # guards the K2 scratch path: a per-call pool release once cost ~10 ms
    import time
    wl = workloads()["c5"]
    dos = isd.DoSHistogram(wl.spec, _golden_c("c5"))
    isd.thermo_grid(dos, wl.fields, wl.temps)
    t0 = time.perf_counter()
    for _ in range(20):
        isd.thermo_grid(dos, wl.fields, wl.temps)
    per_call = (time.perf_counter() - t0) / 20
    assert per_call < 2e-3, per_call
