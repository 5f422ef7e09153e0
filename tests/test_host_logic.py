"""CPU tests of the host side: lattice compiler, C-ABI library, kernel plan.

No GPU: the native library is loaded and its host-only entry points
(isd_validate, isd_plan) are exercised; the hoisted kernel's arithmetic is
replayed in numpy from the plan the library compiles and checked against
the oracle on every configuration.
"""

import ctypes
import os

import numpy as np
import pytest

import paper_1110_2561_b200 as isd
from paper_1110_2561_b200 import _native
from paper_1110_2561_b200.enumeration import native_lattice
from paper_1110_2561_b200.workloads import canonical_ops, workloads
from oracle import naive, port

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# -- library / ABI -----------------------------------------------------------

def test_library_exports_every_header_symbol():
    lib = _native.load()
    header = open(os.path.join(ROOT, "include", "isingdos_b200.h")).read()
    import re
    declared = set(re.findall(r"\b(isd_[a-z_]+)\s*\(", header))
    assert declared == set(_native.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.isd_abi_version() == 2
    assert b"sm_100a" in lib.isd_version()


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.library_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_validate_rejects_bad_lattices():
    good = native_lattice(isd.LatticeSpec(4, 4))
    _native.validate(good)
    bad = _native.make_lattice(16, 31, isd.LatticeSpec(4, 4).bond_classes())
    with pytest.raises(ValueError, match="n_bonds"):
        _native.validate(bad)
    bad = _native.make_lattice(16, 1, [(16, 1, 0)])
    with pytest.raises(ValueError, match="shift"):
        _native.validate(bad)
    bad = _native.make_lattice(16, 1, [(4, 1 << 12, 0)])
    with pytest.raises(ValueError, match="beyond N"):
        _native.validate(bad)
    bad = _native.make_lattice(16, 1, [(1, 1, 2)])
    with pytest.raises(ValueError, match="subset"):
        _native.validate(bad)
    bad = _native.make_lattice(41, 1, [(1, 1, 0)])
    with pytest.raises(ValueError, match="n_spins"):
        _native.validate(bad)


def test_no_gpu_means_loud_failure():
    if _native.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        isd.enumerate_shard(isd.LatticeSpec(2, 2), None,
                            isd.make_shards(isd.LatticeSpec(2, 2), 1)[0])


# -- lattice compiler ----------------------------------------------------------

@pytest.mark.parametrize("spec,expected", [
    (isd.LatticeSpec(5, 5), [(1, 20), (4, 5), (5, 20), (20, 5)]),
    (isd.LatticeSpec(6, 6), [(1, 30), (5, 6), (6, 30), (30, 6)]),
    (isd.LatticeSpec(3, 3, 4),
     [(1, 24), (2, 12), (3, 24), (6, 12), (9, 27), (27, 9)]),
    (isd.LatticeSpec(4, 4, boundary="free"), [(1, 12), (4, 12)]),
    (isd.LatticeSpec(6, 6, boundary="free"), [(1, 30), (6, 30)]),
])
def test_bond_classes_match_survey_appendix_a(spec, expected):
    got = [(s, bin(m).count("1")) for s, m, _ in spec.bond_classes()]
    assert got == expected
    assert sum(c for _, c in got) == spec.num_bonds


LATTICES = [
    dict(rows=2, cols=2), dict(rows=3, cols=3), dict(rows=2, cols=4),
    dict(rows=3, cols=4, coupling=-1), dict(rows=2, cols=2, depth=2),
    dict(rows=2, cols=3, depth=2), dict(rows=3, cols=3, boundary="free"),
    dict(rows=4, cols=4, boundary="free"), dict(rows=2, cols=2, depth=3),
    dict(rows=3, cols=2, depth=2, boundary="free"),
]


def _spec_and_oracle(kw, signed_seed=None):
    spec = isd.LatticeSpec(**kw)
    if signed_seed is not None:
        spec = isd.LatticeSpec(**kw, bond_signs=isd.random_bond_signs(
            spec, signed_seed))
    per = spec.periodic
    signs = list(spec.bond_signs) if spec.bond_signs else None
    return spec, (spec.rows, spec.cols, spec.depth, spec.coupling, per, signs)


@pytest.mark.parametrize("kw", LATTICES)
@pytest.mark.parametrize("seed", [None, 5])
def test_class_energy_equals_per_bond_energy(kw, seed):
    # every index: |J|(2 e_idx - B) == -sum_b J_b s_i s_j (oracle.py:61-63)
    spec, (r, c, d, j, per, signs) = _spec_and_oracle(kw, seed)
    scale = abs(spec.coupling)
    for index in range(spec.num_configs):
        e = scale * (2 * isd.unsatisfied_bonds(spec, index) - spec.num_bonds)
        assert e == naive.energy_of(r, c, d, index, j, per, signs)


def test_total_energy_anchors():
    spec = isd.LatticeSpec(4, 4)
    assert isd.total_energy(isd.decode_config(spec, 0), spec) == -32
    assert isd.total_energy(isd.decode_config(spec, 65535), spec) == -32
    checker = sum(1 << spec.bit_position(r, c)
                  for r in range(4) for c in range(4) if (r + c) % 2)
    assert isd.total_energy(isd.decode_config(spec, checker), spec) == 32
    free = isd.LatticeSpec(4, 4, boundary="free")
    assert isd.total_energy(isd.decode_config(free, 0), free) == -24


def test_latticespec_validation_messages():
    with pytest.raises(ValueError, match="degenerate periodic axis"):
        isd.LatticeSpec(1, 4)
    with pytest.raises(ValueError, match="cap of 40"):
        isd.LatticeSpec(7, 6)
    with pytest.raises(ValueError, match="cap of 30"):
        isd.LatticeSpec(31, 1 + 1)
    with pytest.raises(ValueError, match="coupling"):
        isd.LatticeSpec(2, 2, coupling=0)
    with pytest.raises(ValueError, match="boundary"):
        isd.LatticeSpec(2, 2, boundary="open")
    with pytest.raises(ValueError, match="bond_signs"):
        isd.LatticeSpec(2, 2, bond_signs=(1, -1))
    with pytest.raises(ValueError, match="bond signs"):
        isd.LatticeSpec(2, 2, bond_signs=(2,) * 8)
    assert isd.LatticeSpec(4, 4, 1, 2.0).coupling == 2
    assert isd.LatticeSpec(4, 4) == isd.LatticeSpec(4, 4, 1, 1)
    assert isd.LatticeSpec(4, 4) != isd.LatticeSpec(4, 4, boundary="free")
    assert isd.LatticeSpec(4, 4, boundary="free").num_bonds == 24
    assert isd.LatticeSpec(3, 3, 4).num_bonds == 108


def test_c4_signs_fixture_matches_convention():
    from golden_io import load_json
    fx = load_json("c4_bond_signs.json")
    spec = workloads()["c4"].spec
    assert list(spec.bond_signs) == fx["signs"]
    assert len(fx["signs"]) == 72


def test_canonical_ops_table():
    w = workloads()
    assert [canonical_ops(w[c].spec) for c in ("c1", "c2", "c3", "c4", "c5")] \
        == [(3, 6), (5, 12), (6, 13), (10, 33), (14, 37)]


def test_make_shards_partition():
    spec = isd.LatticeSpec(2, 2)
    assert [s.size for s in isd.make_shards(spec, 3)] == [6, 5, 5]
    big = isd.LatticeSpec(6, 6)
    s8 = isd.make_shards(big, 8)
    assert [s.start_index >> 33 for s in s8] == list(range(8))  # top 3 bits
    with pytest.raises(ValueError):
        isd.make_shards(spec, 17)


# -- hoisted-kernel plan replay ---------------------------------------------

def _u(x):
    return np.uint64(x)


def _band_items(F, n_target, span=2):
    """The host's work-item split of 2^F slots (capi.cu build_band_items)."""
    from math import comb
    cum = [0]
    for q in range(F + 1):
        cum.append(cum[-1] + comb(F, q))
    total = cum[-1]
    size = max(1, -(-total // n_target))
    items, g, q = [], 0, 0
    while g < total:
        while cum[q + 1] <= g:
            q += 1
        g1 = min(g + size, cum[min(F, q + span) + 1])
        items.append((g, g1, q))
        g = g1
    return items, cum


def _slot_rank(v, F, cum):
    """Index of F-bit v in (popcount, value) order."""
    from math import comb
    bits = [b for b in range(F) if (v >> b) & 1]
    return cum[len(bits)] + sum(comb(b, i + 1) for i, b in enumerate(bits))


def replay_hoisted(spec, loop_bits, pair=None, band_items=None,
                   domino=False, band_pair=2):
    """numpy replay of k1_hoisted's arithmetic and address layout.

    Every index is decomposed exactly as the kernel does (run / loop /
    copy sites of the plan), its histogram word is formed from the per-run,
    per-loop and per-copy terms, and the words are read back through the
    kernel's flush rule.  Also asserts the layout is injective on the bins
    that occur and that the e parity formula holds.
    """
    knobs = {"ISD_LOOP_BITS": loop_bits}
    if pair is not None:
        knobs["ISD_PAIR"] = pair
    if band_items is not None:  # force a banded mode-2 plan
        knobs.update(ISD_BAND=1, ISD_PAIR=band_pair,
                     ISD_BAND_LOOP_BITS=loop_bits,
                     ISD_BAND_DOMINO_LOOP_BITS=loop_bits,
                     ISD_BAND_DOMINO=2 if domino else 0)
        if domino:  # lane patterns with domino partners need a "wide" plan
            knobs["ISD_PLAN_WIDE"] = 1
    with _native.knobs(**knobs):
        lat = native_lattice(spec)
        usable, info = _native.plan(lat, spec.num_configs)
    if band_items is not None and (not usable or not info.band_rows or
                                   info.pair_mode != band_pair):
        return None  # no banded layout (of that mode) for this lattice
    assert usable
    if pair == 3 and info.pair_mode != 3:
        return None  # no cluster of three among the low sites
    if pair is not None:
        assert info.pair_mode == pair
    u, k = info.u, info.k
    stride = info.stride
    classes = spec.bond_classes()
    n = spec.num_spins
    above_k = int(info.run_mask_above_k)
    loop = int(info.loop_mask)
    sites = list(info.copy_site)
    copies = sum(1 << q for q in sites)
    assert copies | loop == (1 << k) - 1 and copies & loop == 0
    x = np.arange(1 << n, dtype=np.uint64)
    xt = x & _u(above_k)
    jb = x & _u(loop)
    c = np.zeros(x.shape, dtype=np.int64)
    for t, q in enumerate(sites):
        c |= ((x >> _u(q)) & _u(1)).astype(np.int64) << t
    pc = lambda a: np.bitwise_count(a).astype(np.int64)  # noqa: E731
    m = pc(xt) + pc(jb) + pc(c.astype(np.uint64))
    e = np.zeros(x.shape, dtype=np.int64)
    for s, msk, jn in classes:
        sh = xt >> _u(s)
        e += pc(((xt ^ sh) ^ _u(jn)) & _u(msk) & _u(above_k))
        cst = (sh & _u(0xFFFFFFFF)) ^ _u(jn & 0xFFFFFFFF)
        jshift = (jb >> _u(s)) if s < 32 else np.zeros_like(jb)
        mvar = msk & loop & ~(copies >> s)
        e += pc((jb ^ jshift ^ cst) & _u(mvar))
    n_slot = {}
    for t in range(u):
        nq = pc((xt ^ _u(info.copy_jneg1[t])) & _u(info.copy_nbr1[t]) & _u(above_k))
        nq += pc((xt ^ _u(info.copy_jneg2[t])) & _u(info.copy_nbr2[t]) & _u(above_k))
        nq += pc((jb ^ _u(info.copy_jneg1[t] & loop)) & _u(info.copy_nbr1[t] & loop))
        nq += pc((jb ^ _u(info.copy_jneg2[t] & loop)) & _u(info.copy_nbr2[t] & loop))
        e += nq
        e += np.where((c >> t) & 1, info.copy_degree[t] - 2 * nq, 0)
        n_slot[t] = nq
    kt = np.array(list(info.copy_table), dtype=np.int64)
    e += kt[c] - stride * np.bitwise_count(c.astype(np.uint64)).astype(np.int64)
    A, B, P = info.row_words, info.e_words, info.plane_words
    odd = int(info.odd_mask)
    if info.e_mode:
        par = (pc(x & _u(odd & ~copies)) + info.e_parity) & 1
        assert np.all((e - par) % 2 == 0), "e parity formula"
        word = m * A + ((e - par) // 2) * B + par * P
    else:
        word = m * A + e * B
    key = m * stride + e
    mode = info.pair_mode
    down = np.ones(x.shape, dtype=bool)
    if mode == 3:
        # cluster of three (copy bits 4-6): one RED per configuration with
        # all three down, in the plane of the multiset of their counts
        R, planes = info.pair_degree[0], info.pair_words[1]
        assert planes == (R + 1) * (R + 2) * (R + 3) // 6
        ns = []
        for slot in (u - 3, u - 2, u - 1):
            bit = 1 << slot
            down &= (c & bit) == 0
            # no bond to an unpaired copy site: flipping it changes the
            # copy-copy term only through the cluster's internal bonds
            assert info.copy_degree[slot] == R
            ns.append(n_slot[slot])
        srt = np.sort(np.stack(ns), axis=0)
        lo, mid, hi = srt[0], srt[1], srt[2]
        pat = hi * (hi + 1) * (hi + 2) // 6 + mid * (mid + 1) // 2 + lo
        assert pat[down].min() >= 0 and pat[down].max() < planes
        word = word + pat * info.pair_words[0]
        key = key * planes + pat
    slots = [u - 1, u - 2][:mode] if mode < 3 else []
    for i, slot in enumerate(slots):
        # paired copies: only configurations with the paired copy bits
        # down issue a RED, into pattern plane n + u(c) per paired site
        bit = 1 << slot
        down &= (c & bit) == 0
        cc_deg = info.pair_degree[i] - info.copy_degree[slot]
        u_c = (cc_deg - (kt[c | bit] - kt[c & ~bit] - stride)) // 2
        pat = n_slot[slot] + u_c
        word = word + pat * info.pair_words[i]
        key = key * (info.pair_degree[i] + 1) + pat
        assert pat[down].min() >= 0 and pat[down].max() <= info.pair_degree[i]
    if info.band_rows:
        # banded: each run's slot (its non-pivot run bits) falls in a work
        # item whose base row q0 the table rows are relative to
        run = (x >> _u(k)).astype(np.int64)
        rb = n - k
        pivots = int(info.lane_mask)
        # lane bit i = the run's bit at pivot i; XOR the lane pattern (with
        # any domino partners) out to get the warp's slot bits
        for v in info.lane_vec:
            piv = int(v) & pivots
            assert piv and piv & (piv - 1) == 0
            run = run ^ (((run & piv) != 0) * (int(v) & ~piv))
        free = [b for b in range(rb) if not (pivots >> b) & 1]
        F = len(free)
        items, cum = _band_items(F, band_items, span=int(info.band_span))
        starts = np.array([it[0] for it in items], dtype=np.int64)
        vals = np.zeros(run.shape, dtype=np.int64)
        for j, b in enumerate(free):
            vals |= ((run >> b) & 1) << j
        uniq, inv = np.unique(vals, return_inverse=True)
        gidx = np.array([_slot_rank(int(v), F, cum) for v in uniq])[inv]
        item_of = np.searchsorted(starts, gidx, side="right") - 1
        q0 = np.array([it[2] for it in items], dtype=np.int64)[item_of]
        row = m - q0
        assert row.min() >= 0 and row[down].max() < info.band_rows
        word = word - q0 * A
        key = key + 0
    word, key = word[down], key[down]
    assert word.max() < info.hist_words
    if info.band_rows:
        return _banded_table(info, spec, word, key, item_of[down],
                             q0[down], len(items), odd, A, B, P)
    # injective on occurring bins
    pairs = np.unique(np.stack([word, key]), axis=1)
    assert len(np.unique(pairs[0])) == pairs.shape[1], "layout collision"
    hist = np.bincount(word, minlength=int(info.hist_words))

    def bin_word(mm, ee):
        if info.e_mode:
            p2 = ee & 1
            return mm * A + ((ee - p2) // 2) * B + p2 * P
        return mm * A + ee * B

    srcs = _flush_sources(info)
    table = np.zeros((n + 1, stride), dtype=np.int64)
    for mm in range(n + 1):
        for ee in range(stride):
            if info.e_mode and odd == 0 and (ee & 1) != info.e_parity:
                continue
            tot = 0
            for plane, dr, de in srcs:
                sm, se = mm - dr, ee - de
                if sm >= 0 and 0 <= se < stride:
                    tot += hist[bin_word(sm, se) + plane]
            table[mm, ee] = tot
    return table


def _flush_sources(info):
    """(plane word offset, rows up, e shift) of every source word of a bin:
    the kernel's flush rule per pairing mode."""
    mode = info.pair_mode
    D, S = list(info.pair_degree), list(info.pair_words)
    if mode == 0:
        return [(0, 0, 0)]
    srcs = []
    if mode == 3:
        R, i1, idx = D[0], info.pair_both, 0
        for cc in range(R + 1):
            for bb in range(cc + 1):
                for aa in range(bb + 1):
                    f = [R - 2 * aa, R - 2 * bb, R - 2 * cc]
                    for sub in range(8):
                        j = bin(sub).count("1")
                        de = sum(f[i] for i in range(3) if (sub >> i) & 1)
                        de += i1 if j in (1, 2) else 0
                        srcs.append((idx * S[0], j, de))
                    idx += 1
        return srcs
    for p1 in range(D[1] + 1 if mode == 2 else 1):
        for p0 in range(D[0] + 1):
            plane = p0 * S[0] + (p1 * S[1] if mode == 2 else 0)
            f0, f1 = D[0] - 2 * p0, D[1] - 2 * p1
            srcs += [(plane, 0, 0), (plane, 1, f0)]
            if mode == 2:
                srcs += [(plane, 1, f1), (plane, 2, f0 + f1 + info.pair_both)]
    return srcs


def _banded_table(info, spec, word, key, item, q0, n_items, odd, A, B, P):
    """Per-item tables and the kernel's banded mode-2 flush rule."""
    n, stride = spec.num_spins, info.stride
    R = info.band_rows
    srcs = _flush_sources(info)

    def bin_word(rr, ee):
        if info.e_mode:
            p2 = ee & 1
            return rr * A + ((ee - p2) // 2) * B + p2 * P
        return rr * A + ee * B

    table = np.zeros((n + 1, stride), dtype=np.int64)
    for it in range(n_items):
        sel = item == it
        if not sel.any():
            continue
        w, kk = word[sel], key[sel]
        pairs = np.unique(np.stack([w, kk]), axis=1)
        assert len(np.unique(pairs[0])) == pairs.shape[1], "layout collision"
        hist = np.bincount(w, minlength=int(info.hist_words))
        base = int(q0[sel][0])
        assert (q0[sel] == base).all()
        for mm in range(base, min(n, base + R + info.pair_mode - 1) + 1):
            for ee in range(stride):
                if info.e_mode and odd == 0 and (ee & 1) != info.e_parity:
                    continue
                tot = 0
                for plane, dr, de in srcs:
                    rr, se = mm - base - dr, ee - de
                    if 0 <= rr < R and 0 <= se < stride:
                        tot += hist[bin_word(rr, se) + plane]
                table[mm, ee] += tot
    return table


REPLAY = [
    dict(rows=4, cols=4), dict(rows=3, cols=4, coupling=-1),
    dict(rows=2, cols=2, depth=3), dict(rows=4, cols=4, boundary="free"),
    dict(rows=2, cols=4, depth=2), dict(rows=3, cols=3, depth=2),
    dict(rows=5, cols=3), dict(rows=2, cols=8),
    dict(rows=4, cols=3, boundary="free"), dict(rows=3, cols=5, boundary="free"),
    dict(rows=2, cols=3, depth=2, boundary="free"),
]


@pytest.mark.parametrize("kw", REPLAY)
@pytest.mark.parametrize("seed", [None, 11])
@pytest.mark.parametrize("loop_bits", [0, 3, 7])
@pytest.mark.parametrize("pair", [0, 1, 2, 3])
def test_hoisted_plan_replay_matches_oracle(kw, seed, loop_bits, pair):
    spec, (r, c, d, j, per, signs) = _spec_and_oracle(kw, seed)
    if spec.num_spins < 7 + loop_bits + 1:
        pytest.skip("lattice too small for this loop width")
    lat = port.Lattice(r, c, d, j, per, signs)
    want = port.enumerate_range(lat, 0, 1 << lat.n)
    got = replay_hoisted(spec, loop_bits, pair)
    if got is None:
        pytest.skip("no cluster of three like sites in the low bits")
    assert np.array_equal(got, want)


BAND_REPLAY = [dict(rows=4, cols=4), dict(rows=2, cols=3, depth=3),
               dict(rows=5, cols=4), dict(rows=4, cols=5, boundary="free"),
               dict(rows=3, cols=3, depth=2)]


@pytest.mark.parametrize("kw", BAND_REPLAY)
@pytest.mark.parametrize("seed", [None, 11])
@pytest.mark.parametrize("n_items", [3, 17])
@pytest.mark.parametrize("domino", [False, True])
@pytest.mark.parametrize("band_pair", [2, 3])
def test_banded_plan_replay_matches_oracle(kw, seed, n_items, domino,
                                           band_pair):
    # banded mode 2: per-item tables of band_rows rows, the kernel's slot
    # order and item split replayed, flushed per item, against the oracle;
    # both band shapes (single-site lanes; domino lanes, one popcount class
    # per item)
    spec, (r, c, d, j, per, signs) = _spec_and_oracle(kw, seed)
    # (a cluster of three plus four sites adjacent to none of them needs
    # more low sites than the 8 of a one-site loop)
    got = replay_hoisted(spec, 1 if band_pair == 2 else 4,
                         band_items=n_items, domino=domino,
                         band_pair=band_pair)
    if got is None:
        pytest.skip("no banded layout")
    lat = port.Lattice(r, c, d, j, per, signs)
    assert np.array_equal(got, port.enumerate_range(lat, 0, 1 << lat.n))


TRI_REPLAY = [dict(rows=3, cols=3, depth=2), dict(rows=3, cols=6),
              dict(rows=3, cols=6, coupling=-1), dict(rows=6, cols=3)]


@pytest.mark.parametrize("kw", TRI_REPLAY)
@pytest.mark.parametrize("seed", [None, 11])
@pytest.mark.parametrize("banded", [None, 3, 17])
def test_cluster_plan_replay_matches_oracle(kw, seed, banded):
    # pair mode 3 on lattices with a periodic axis of length 3 (a triangle of
    # mutually adjacent sites, as c5 has): multiset planes, 8 configurations
    # per RED, unbanded and banded, uniform and +-J bonds
    spec, (r, c, d, j, per, signs) = _spec_and_oracle(kw, seed)
    if banded is None:
        got = replay_hoisted(spec, 5, pair=3)
    else:
        got = replay_hoisted(spec, 5, band_items=banded, band_pair=3)
    if got is None:
        pytest.skip("no cluster plan")
    lat = port.Lattice(r, c, d, j, per, signs)
    assert np.array_equal(got, port.enumerate_range(lat, 0, 1 << lat.n))


def test_c5_cluster_plan():
    # c5 (3x3x4): the banded cluster plan pairs the x-row (9, 10, 11) of
    # layer 1 — four external bonds each, 35 multiset planes — with four
    # unpaired copy sites among sites 3..8
    spec = workloads()["c5"].spec
    with _native.knobs(ISD_PAIR=3, ISD_BAND=1):
        usable, info = _native.plan(native_lattice(spec), spec.num_configs)
    assert usable and info.pair_mode == 3 and info.band_rows > 0
    assert sorted(info.copy_site[4:]) == [9, 10, 11]
    assert all(3 <= q <= 8 for q in info.copy_site[:4])
    assert info.pair_degree[0] == 4 and info.pair_words[1] == 35
    assert info.pair_both == 2 and info.hist_words * 4 <= 227 * 1024


def test_plan_copy_site_variants(monkeypatch):
    for name in ("c5", "c4"):  # periodic: every site has even degree
        spec = workloads()[name].spec
        usable, info = _native.plan(native_lattice(spec), spec.num_configs)
        assert usable and info.e_mode == 1 and info.odd_mask == 0
    _native.set_knob("ISD_COPY_VARIANT", "even")
    spec = workloads()["c3"].spec
    usable, info = _native.plan(native_lattice(spec), spec.num_configs)
    assert usable and info.e_mode == 1
    assert info.odd_mask != 0 and info.plane_words > 0
    assert all(not (int(info.odd_mask) >> q) & 1 for q in info.copy_site)
    _native.set_knob("ISD_COPY_VARIANT", "low")
    usable, info = _native.plan(native_lattice(spec), spec.num_configs)
    assert usable and info.e_mode == 0
    assert sorted(info.copy_site) == list(range(7))


def test_plan_refuses_tiny_lattices():
    usable, _ = _native.plan(native_lattice(isd.LatticeSpec(2, 2)), 16)
    assert not usable


def _integration_stub_classes(spec):
    # the class compiler shown in INTEGRATION.md (a reference-side binding)
    R, C, D = spec.rows, spec.cols, spec.depth
    dims, strides = (R, C, D), (1, R, R * C)
    out = []
    for a in range(3 if D > 1 else 2):
        inner = wrap = 0
        for l in range(D):
            for c in range(C):
                for r in range(R):
                    coord = (r, c, l)[a]
                    bit = 1 << ((l * C + c) * R + r)
                    if coord < dims[a] - 1:
                        inner |= bit
                    if coord == 0:
                        wrap |= bit
        neg = spec.coupling < 0
        out += [(strides[a], inner, inner if neg else 0),
                ((dims[a] - 1) * strides[a], wrap, wrap if neg else 0)]
    return out


@pytest.mark.parametrize("spec", [isd.LatticeSpec(4, 4), isd.LatticeSpec(5, 5),
                                  isd.LatticeSpec(3, 3, 4),
                                  isd.LatticeSpec(2, 3, 2, -1),
                                  isd.LatticeSpec(17, 2)])
def test_integration_stub_matches_bond_classes(spec):
    assert _integration_stub_classes(spec) == spec.bond_classes()


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_jit_source_compiles_for_sm100a(name):
    # the per-lattice specialised kernel is generated and NVRTC-compiled on
    # the host (no GPU needed); a compile error would silently cost speed
    spec = workloads()[name].spec
    n = _native.jit_check(native_lattice(spec), spec.num_configs)
    assert n > 10000


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
@pytest.mark.parametrize("log_hint", [33, 34, 36])
def test_lane_patterns_tile_the_walk(name, log_hint):
    # every lane vector has its own pivot, and all of them stay inside the
    # run bits a walk of 2^log_hint configurations varies (shards of an
    # 8-GPU run use log_hint = 33)
    spec = workloads()[name].spec
    usable, info = _native.plan(native_lattice(spec), 1 << log_hint)
    assert usable
    mask = int(info.lane_mask)
    vecs = [int(v) for v in info.lane_vec]
    assert bin(mask).count("1") == 5
    assert sorted(v & mask for v in vecs) == sorted(1 << b for b in range(64)
                                                   if (mask >> b) & 1)
    span = 0
    for v in vecs + [mask]:
        span = max(span, v.bit_length())
    assert span <= log_hint - info.k


# The host's work-item split of banded launches (capi.cu -> plan.cpp
# band_work_items, exported as isd_band_items for this test): items tile the
# slot order, stay within span + 1 popcount classes, and with the small
# items of the extreme classes added to blocks 0 and 1 every block gets the
# same cost.
@pytest.mark.parametrize("F,n_target", [(19, 148), (16, 148), (12, 37),
                                        (8, 7)])
@pytest.mark.parametrize("weighted", [False, True])
def test_band_items_tile_and_balance(F, n_target, weighted):
    from bisect import bisect_right
    from math import comb
    rng = np.random.default_rng(F * 1000 + n_target)
    n_seg = min(1 << F, 2048) if weighted else 0
    w = 1.0 + 0.8 * rng.random(n_seg) if weighted else None
    flush = 20.0
    items, exact = _native.band_items(F, n_target, 2, w, flush)
    cum = [0]
    for q in range(F + 1):
        cum.append(cum[-1] + comb(F, q))
    cls = lambda g: bisect_right(cum, g) - 1  # noqa: E731
    r = items[np.argsort(items[:, 0])]
    assert r[0, 0] == 0 and r[-1, 1] == 1 << F
    assert np.array_equal(r[1:, 0], r[:-1, 1]) and np.all(r[:, 1] > r[:, 0])
    for g0, g1, q0 in items:
        assert cls(g0) == q0 and cls(g1 - 1) <= q0 + 2

    total = 1 << F
    seg = np.arange(total) * max(n_seg, 1) // total
    per_slot = w[seg] if weighted else np.ones(total)
    csum = np.concatenate([[0.0], np.cumsum(per_slot)])
    cost = [csum[g1] - csum[g0] for g0, g1, _ in items]
    if not exact:
        assert F <= 12  # class caps bind on small walks: plain split
        return
    block = np.array(cost[:n_target])
    for i, c in enumerate(cost[n_target:]):
        block[i] += c + flush  # a second item costs its walk and a flush
    assert len(items) >= n_target
    assert block.max() <= 1.01 * block.mean() + 2 * per_slot.max()
    assert block.min() >= 0.99 * block.mean() - 2 * per_slot.max()


def test_band_items_valid_for_every_walk_size():
    # tiny walks (a flush outweighs an item) through full-size ones, every
    # block count, flush cost and cost curve: always a tiling of the slot
    # order with non-empty items inside their class span
    from bisect import bisect_right
    from math import comb
    for F in range(1, 20):
        cum = [0]
        for q in range(F + 1):
            cum.append(cum[-1] + comb(F, q))
        for nt in (1, 3, 7, 148):
            for flush in (0.0, 78.0, 312.0, 5000.0):
                for weighted in (False, True):
                    w = (np.linspace(1, 2, min(1 << F, 9472)) if weighted
                         else None)
                    items, _ = _native.band_items(F, nt, 2, w, flush)
                    r = items[np.argsort(items[:, 0])]
                    assert r[0, 0] == 0 and r[-1, 1] == 1 << F
                    assert np.array_equal(r[1:, 0], r[:-1, 1])
                    assert np.all(r[:, 1] > r[:, 0])
                    for g0, g1, q0 in items:
                        assert bisect_right(cum, g0) - 1 == q0
                        assert bisect_right(cum, g1 - 1) - 1 <= q0 + 2


@pytest.mark.parametrize("R,I1", [(4, 2), (4, 0), (5, -2), (6, 0)])
def test_cluster_flush_folded_sums_equal_direct_gather(R, I1):
    # k1_body.cuh, PAIR == 3, specialised build: the two-stage flush folds
    # the multiset planes of a cell into G0, G1[v], G2[t], G3[t] and gathers
    # 6R + 4 shifted sums per bin; it must equal the direct gather of 8
    # shifted words per plane (one per subset of the cluster flipped up)
    rng = np.random.default_rng(R * 10 + I1)
    rows, ncol = 9, 40
    planes = [(a, b, c) for c in range(R + 1) for b in range(c + 1)
              for a in range(b + 1)]
    H = {p: rng.integers(0, 1000, size=(rows, ncol)) for p in planes}

    def at(arr, r, e):
        return int(arr[r, e]) if 0 <= r < rows and 0 <= e < ncol else 0

    direct = np.zeros((rows + 3, ncol), dtype=np.int64)
    for r in range(rows + 3):
        for e in range(ncol):
            s = 0
            for (a, b, c), h in H.items():
                f = [R - 2 * a, R - 2 * b, R - 2 * c]
                s += at(h, r, e)
                for i in range(3):
                    s += at(h, r - 1, e - f[i] - I1)
                for i in range(3):
                    for j in range(i + 1, 3):
                        s += at(h, r - 2, e - f[i] - f[j] - I1)
                s += at(h, r - 3, e - sum(f))
            direct[r, e] = s
    g0 = sum(H.values())
    g1 = [sum(h * p.count(v) for p, h in H.items()) for v in range(R + 1)]
    g2 = [sum(h * sum(1 for i in range(3) for j in range(i + 1, 3)
                      if p[i] + p[j] == t) for p, h in H.items())
          for t in range(2 * R + 1)]
    g3 = [sum((h for p, h in H.items() if sum(p) == t),
              np.zeros((rows, ncol), dtype=np.int64))
          for t in range(3 * R + 1)]
    folded = np.zeros_like(direct)
    for r in range(rows + 3):
        for e in range(ncol):
            s = at(g0, r, e)
            s += sum(at(g1[v], r - 1, e - (R - 2 * v) - I1)
                     for v in range(R + 1))
            s += sum(at(g2[t], r - 2, e - (2 * R - 2 * t) - I1)
                     for t in range(2 * R + 1))
            s += sum(at(g3[t], r - 3, e - (3 * R - 2 * t))
                     for t in range(3 * R + 1))
            folded[r, e] = s
    assert np.array_equal(direct, folded)
    assert 6 * R + 4 <= len(planes)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
@pytest.mark.parametrize("log_hint", [33, 36])
def test_band_slot_order_is_a_permutation_of_the_free_run_bits(name, log_hint):
    # capi.cu band_slot_order / k1_body.cuh IsdSlotMap: slot bit i lands on
    # run bit pos[i]; any order must be a bijection onto the run bits that
    # are not lane pivots (every run is then walked exactly once), and the
    # natural order is the increasing one
    from paper_1110_2561_b200 import _native
    from paper_1110_2561_b200.enumeration import native_lattice
    from paper_1110_2561_b200.workloads import workloads
    spec = workloads()[name].spec
    lat = native_lattice(spec)
    _native.set_knob("ISD_BAND", "1")
    _native.set_knob("ISD_PAIR", "3")
    ok, plan = _native.plan(lat, 1 << log_hint)
    if not plan.band_rows:
        pytest.skip("no banded plan")
    run_bits = log_hint - plan.k
    free = [b for b in range(run_bits) if not (plan.lane_mask >> b) & 1]
    natural = list(_native.band_slot_order(lat, plan, 0, run_bits, False))
    assert natural == free
    ordered = list(_native.band_slot_order(lat, plan, 0, run_bits, True))
    assert sorted(ordered) == free
    # deterministic (fixed seed): the same plan gives the same order
    assert ordered == list(_native.band_slot_order(lat, plan, 0, run_bits, True))
