"""Seeded lattice-shape fuzz: the B200 engine vs the C oracle.

The fixed-shape parity tests cover the reference goldens and BASELINE's
five lattices; this file draws many more geometries (2D and 3D, axes of
length 2 with their double bonds, free edges, +/-J, negative and
non-integral J) from a fixed seed and compares

* whole tables (N <= 22) walked by `full_dos` with the C oracle's full walk;
* random slices (N up to 40) walked through `enumerate_range_timed` with the
  C oracle on the same [start, end).

The oracle side builds its bond list from the naive oracle's geometry
(oracle/naive.py), so it shares no code with the product's bond compiler.
Bit-exact equality is required.
"""

import os
import random

import numpy as np
import pytest

import paper_1110_2561_b200 as isd
from paper_1110_2561_b200 import _native
from paper_1110_2561_b200.enumeration import enumerate_range_timed
from oracle import cref

pytestmark = pytest.mark.gpu

COUPLINGS = (1, -1, 0.5, -2.5, 3)


def draw_specs(seed, count, n_lo, n_hi):
    """`count` random valid lattices with n_lo <= N <= n_hi."""
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        rows = rng.randint(2, 12)
        cols = rng.randint(2, 12)
        depth = rng.choice((1, 1, 2, 3, 4))
        n = rows * cols * depth
        if not n_lo <= n <= n_hi:
            continue
        kw = dict(boundary=rng.choice(("periodic", "free")))
        spec = isd.LatticeSpec(rows, cols, depth, rng.choice(COUPLINGS), **kw)
        if rng.random() < 0.4:
            spec = isd.LatticeSpec(rows, cols, depth, spec.coupling, **kw,
                                   bond_signs=isd.random_bond_signs(
                                       spec, rng.randrange(1 << 30)))
        out.append(spec)
    return out


def oracle_table(spec, start=0, end=None):
    return cref.table(spec.rows, spec.cols, spec.depth, spec.coupling,
                      spec.periodic,
                      list(spec.bond_signs) if spec.bond_signs else None,
                      mode="mask", start=start, end=end)


WHOLE = draw_specs(20261020, 120, 4, 22)
SLICED = draw_specs(1110_2561, 60, 23, 40)


@pytest.mark.parametrize("spec", WHOLE, ids=repr)
def test_whole_table_matches_c_oracle(spec):
    got = isd.full_dos(spec)
    want = oracle_table(spec)
    assert np.array_equal(got.counts, want)
    assert isd.verify_dos(got).passed


@pytest.mark.parametrize("spec", SLICED, ids=repr)
def test_slices_match_c_oracle(spec):
    rng = random.Random(spec.num_spins * 7919 + spec.num_bonds)
    for _ in range(3):
        size = rng.choice((1, 977, 1 << 16, (1 << 20) + 3))
        start = rng.randrange(0, spec.num_configs - size)
        table, _ = enumerate_range_timed(spec, start, start + size)
        assert np.array_equal(table.view(np.int64),
                              oracle_table(spec, start, start + size)), start


# The NVRTC-specialised kernel (normally only for walks >= 2^33) walks the
# lowest 1-5 loop sites in Gray order, updating e and the copy-site counts
# per flip; force it (ISD_JIT=2), a loop width, each Gray level and each
# pairing mode on lattices of every kind, against the C oracle.
JIT_SPECS = [s for s in WHOLE if s.num_spins >= 14][:8]


@pytest.mark.parametrize("gray", ["1", "2", "3", "4", "5"])
@pytest.mark.parametrize("pair", ["0", "1", "2", "3"])
@pytest.mark.parametrize("spec", JIT_SPECS, ids=repr)
def test_jit_gray_walk_matches_c_oracle(spec, pair, gray, monkeypatch):
    # Gray widths 3-5 unroll 2^G copies of the RED tree: on 4 lattices, not
    # unpaired beyond G = 3 (4096 REDs of code), and not through the
    # bounds-checked build (its NVRTC compile of G = 5 takes minutes)
    if int(gray) >= 3:
        if JIT_SPECS.index(spec) >= 4 or (pair == "0" and int(gray) >= 4):
            pytest.skip("Gray width >= 3: a subset of the lattices and modes")
        if os.environ.get("ISD_LIBRARY", "").endswith("_dbg.so"):
            pytest.skip("Gray width >= 3 runs through the release build")
    _native.set_knob("ISD_JIT", "2")
    _native.set_knob("ISD_LOOP_BITS", "5" if gray == "5" else "4")
    _native.set_knob("ISD_GRAY", gray)
    _native.set_knob("ISD_PAIR", pair)
    if pair == "3":  # (a cluster of three needs more low sites: l = 5)
        from paper_1110_2561_b200.enumeration import native_lattice
        _native.set_knob("ISD_LOOP_BITS", "5")
        _, info = _native.plan(native_lattice(spec), spec.num_configs)
        if info.pair_mode != 3:
            pytest.skip("no cluster of three like sites in the low bits")
    got = isd.full_dos(spec)
    assert _native_kernel_path().startswith("k1_hoisted_jit")
    assert np.array_equal(got.counts, oracle_table(spec))


def _native_kernel_path():
    from paper_1110_2561_b200 import _native
    return _native.kernel_info()


# Banded mode-2 tables (c5's layout: rows of m relative to each work
# item's base, work items of run slots in popcount order): forced on small
# lattices through both kernel builds, against the C oracle.
@pytest.mark.parametrize("jit", ["0", "2"])
@pytest.mark.parametrize("loop_bits", ["1", "3"])
@pytest.mark.parametrize("pair", ["2", "3"])
@pytest.mark.parametrize("spec", JIT_SPECS, ids=repr)
def test_banded_walk_matches_c_oracle(spec, pair, loop_bits, jit, monkeypatch):
    from paper_1110_2561_b200 import _native
    from paper_1110_2561_b200.enumeration import native_lattice
    if pair == "3":  # (a cluster of three needs more low sites)
        loop_bits = str(int(loop_bits) + 3)
    _native.set_knob("ISD_PAIR", pair)
    _native.set_knob("ISD_BAND", "1")
    _native.set_knob("ISD_BAND_LOOP_BITS", loop_bits)
    _native.set_knob("ISD_JIT", jit)
    _native.set_knob("ISD_LOOP_BITS", loop_bits)
    _, info = _native.plan(native_lattice(spec), spec.num_configs)
    if (not info.band_rows or spec.num_spins - info.k < 6 or
            info.pair_mode != int(pair)):
        pytest.skip("no banded plan for this lattice")
    got = isd.full_dos(spec)
    assert np.array_equal(got.counts, oracle_table(spec))


# Pair mode 3 (a cluster of three like sites: 8 configurations per RED,
# multiset pattern planes) on lattices with a periodic axis of length 3 (a
# triangle of mutually adjacent sites, as c5 has) and on ones where the
# cluster is three non-adjacent sites: both kernel builds, unbanded and
# banded tables, against the C oracle.
TRI_SPECS = [
    isd.LatticeSpec(3, 3, 2), isd.LatticeSpec(3, 6), isd.LatticeSpec(3, 7, 1, -1),
    isd.LatticeSpec(6, 3), isd.LatticeSpec(3, 3, 2, 1, boundary="free"),
    isd.LatticeSpec(5, 4), isd.LatticeSpec(4, 5, boundary="free"),
    isd.LatticeSpec(3, 6, 1, 1, bond_signs=isd.random_bond_signs(
        isd.LatticeSpec(3, 6), 77)),
    isd.LatticeSpec(5, 4, 1, 1, bond_signs=isd.random_bond_signs(
        isd.LatticeSpec(5, 4), 78)),
]


@pytest.mark.parametrize("jit", ["0", "2"])
@pytest.mark.parametrize("band", ["0", "1"])
@pytest.mark.parametrize("loop_bits", ["4", "5"])
@pytest.mark.parametrize("spec", TRI_SPECS, ids=repr)
def test_cluster_walk_matches_c_oracle(spec, loop_bits, band, jit):
    from paper_1110_2561_b200.enumeration import native_lattice
    _native.set_knob("ISD_PAIR", "3")
    _native.set_knob("ISD_BAND", band)
    _native.set_knob("ISD_BAND_LOOP_BITS", loop_bits)
    _native.set_knob("ISD_LOOP_BITS", loop_bits)
    _native.set_knob("ISD_JIT", jit)
    _, info = _native.plan(native_lattice(spec), spec.num_configs)
    if info.pair_mode != 3 or bool(info.band_rows) != (band == "1") or (
            info.band_rows and spec.num_spins - info.k < 6):
        pytest.skip("no such cluster plan for this lattice")
    got = isd.full_dos(spec)
    assert np.array_equal(got.counts, oracle_table(spec))
    assert isd.verify_dos(got).passed


# Mirrored work items (the item's table holds its rows in descending order,
# chosen per item by the bank-conflict model): forced off, per item, and on
# for every item, in banded modes 2 and 3 and both kernel builds.
@pytest.mark.parametrize("jit", ["0", "2"])
@pytest.mark.parametrize("mirror", ["0", "1", "2"])
@pytest.mark.parametrize("pair", ["2", "3"])
@pytest.mark.parametrize("spec", [TRI_SPECS[0], TRI_SPECS[1], TRI_SPECS[5],
                                  TRI_SPECS[7]], ids=repr)
def test_mirrored_band_items_match_c_oracle(spec, pair, mirror, jit):
    from paper_1110_2561_b200.enumeration import native_lattice
    lb = "5" if pair == "3" else "3"
    _native.set_knob("ISD_PAIR", pair)
    _native.set_knob("ISD_BAND", "1")
    _native.set_knob("ISD_BAND_LOOP_BITS", lb)
    _native.set_knob("ISD_LOOP_BITS", lb)
    _native.set_knob("ISD_BAND_MIRROR", mirror)
    _native.set_knob("ISD_JIT", jit)
    _, info = _native.plan(native_lattice(spec), spec.num_configs)
    if (not info.band_rows or spec.num_spins - info.k < 6 or
            info.pair_mode != int(pair)):
        pytest.skip("no banded plan for this lattice")
    got = isd.full_dos(spec)
    assert np.array_equal(got.counts, oracle_table(spec))


# Large aligned shards through the default path (autotuned plan, NVRTC
# kernel, banded mode-3 tables with mirrored items in influence order,
# calibrated cuts) on lattices outside the BASELINE set: one 2^33-
# configuration shard each, bit-exact against the C oracle's walk of the
# same range.
LARGE_SHARDS = [
    (isd.LatticeSpec(5, 7), 3),
    (isd.LatticeSpec(2, 17, boundary="free"), 1),
    (isd.LatticeSpec(4, 9, 1, -1), 5),
    (isd.LatticeSpec(3, 4, 3, 1, bond_signs=isd.random_bond_signs(
        isd.LatticeSpec(3, 4, 3), 4242)), 6),
    (isd.LatticeSpec(6, 6, 1, 1, boundary="free",
                     bond_signs=isd.random_bond_signs(
                         isd.LatticeSpec(6, 6, boundary="free"), 99)), 2),
    (isd.LatticeSpec(3, 3, 4), 5),
]


@pytest.mark.parametrize("spec,index", LARGE_SHARDS,
                         ids=[repr(s) for s, _ in LARGE_SHARDS])
def test_large_aligned_shard_matches_c_oracle(spec, index):
    size = 1 << 33
    start = index * size
    assert start + size <= spec.num_configs
    got, _ = enumerate_range_timed(spec, start, start + size)
    assert _native.kernel_info().startswith("k1_hoisted")
    want = oracle_table(spec, start, start + size)
    assert np.array_equal(got.view(np.int64), want)
