"""Semantics of the public API, following the reference's test strategy
(lattice, enumeration and thermodynamics unit tests).

CPU tests cover the host-side value types and scalar helpers; `gpu` tests
cover the properties the reference checks on whole tables (antiferromagnet
mirror, merge, limits of Z, field symmetry, ...), here computed by the
B200 engine.
"""

import math
import random

import numpy as np
import pytest

import paper_1110_2561_b200 as isd
import paper_1110_2561_b200.crosscheck  # noqa: F401  (isd.crosscheck)
from golden_io import read_csv_table


# -- lattice (CPU) ------------------------------------------------------------

@pytest.mark.parametrize("dims", [(2, 2, 1), (2, 3, 1), (3, 3, 1), (2, 2, 2),
                                  (4, 4, 1)])
def test_decode_encode_round_trip(dims):
    spec = isd.LatticeSpec(*dims)
    for index in range(spec.num_configs):
        cfg = isd.decode_config(spec, index)
        assert len(cfg.words) == spec.num_words
        assert all(0 <= w <= spec.word_mask for w in cfg.words)
        assert isd.encode_words(spec, cfg.words) == index


def test_decode_encode_rejections():
    spec = isd.LatticeSpec(2, 2)
    for bad in (-1, 16):
        with pytest.raises(ValueError):
            isd.decode_config(spec, bad)
    with pytest.raises(ValueError, match="stray"):
        isd.encode_words(spec, (0b100, 0))
    with pytest.raises(ValueError):
        isd.encode_words(spec, (0,))


def test_tables_and_popcount():
    t = isd.build_tables(6)
    assert len(t.popcount_table) == 64 and len(t.shift_table) == 64
    for w in range(64):
        assert t.popcount_table[w] == isd.popcount(w) == bin(w).count("1")
        assert t.shift_table[w] == isd.circular_shift(w, 6)
    assert isd.popcount((1 << 40) - 1) == 40
    with pytest.raises(ValueError, match="16"):
        isd.build_tables(17)
    with pytest.raises(ValueError):
        isd.build_tables(1)


def test_word_bond_kernels():
    t = isd.build_tables(4)
    assert isd.aligned_row_bonds(0b0110, 0b0110, t) == 4
    assert isd.aligned_row_bonds(0b0110, 0b1001, t) == 0
    assert isd.aligned_column_bonds(0b0000, t) == 4
    assert isd.aligned_column_bonds(0b0101, t) == 0
    t2 = isd.build_tables(2)  # ring of two: the double bond
    assert isd.aligned_column_bonds(0b00, t2) == 2
    assert isd.aligned_column_bonds(0b10, t2) == 0


def _all_up(spec):
    return isd.decode_config(spec, spec.num_configs - 1)


@pytest.mark.parametrize("dims", [(2, 2, 1), (3, 4, 1), (2, 2, 3), (3, 3, 2)])
def test_uniform_ground_states(dims):
    spec = isd.LatticeSpec(*dims)
    for cfg in (_all_up(spec), isd.decode_config(spec, 0)):
        assert isd.total_energy(cfg, spec) == -spec.num_bonds
    anti = isd.LatticeSpec(*dims, coupling=-1)
    assert isd.total_energy(_all_up(anti), anti) == anti.num_bonds


@pytest.mark.parametrize("kw", [dict(rows=4, cols=4), dict(rows=3, cols=4),
                                dict(rows=2, cols=3, depth=2),
                                dict(rows=4, cols=4, boundary="free")])
def test_flip_and_translation_invariance(kw):
    spec = isd.LatticeSpec(**kw)
    rng = random.Random(23)
    full = spec.num_configs - 1
    for _ in range(150):
        x = rng.randrange(spec.num_configs)
        cfg = isd.decode_config(spec, x)
        m, e = isd.spin_excess(cfg, spec), isd.total_energy(cfg, spec)
        flip = isd.decode_config(spec, x ^ full)
        assert isd.spin_excess(flip, spec) == -m
        assert isd.total_energy(flip, spec) == e
        if spec.periodic:
            rolled = [isd.circular_shift(w, spec.rows) for w in cfg.words]
            r = isd.decode_config(spec, isd.encode_words(spec, rolled))
            assert (isd.spin_excess(r, spec), isd.total_energy(r, spec)) == (m, e)


def test_table_and_direct_energy_paths_agree():
    spec = isd.LatticeSpec(3, 4)
    t = isd.build_tables(3)
    for index in range(spec.num_configs):
        cfg = isd.decode_config(spec, index)
        assert isd.total_energy(cfg, spec, None) == isd.total_energy(cfg, spec, t)


def test_histogram_index_maps():
    spec = isd.LatticeSpec(3, 4, coupling=0.5)
    h = isd.DoSHistogram(spec)
    assert h.m_index(12) == 12 and h.m_index(-12) == 0
    assert h.e_index(-12.0) == 0 and h.e_value(24) == 12.0
    with pytest.raises(ValueError):
        h.m_index(3)
    with pytest.raises(ValueError):
        h.e_index(0.25)
    assert h.count(3, 0) == 0
    with pytest.raises(ValueError):
        isd.DoSHistogram(spec, np.zeros((2, 2)))


def test_merge_and_add():
    rows, cols, depth, j, table = read_csv_table("dos_3x3x1_J1.csv")
    spec = isd.LatticeSpec(rows, cols, depth, j)
    a = isd.DoSHistogram(spec, table // 2)
    b = isd.DoSHistogram(spec, table - table // 2)
    assert isd.merge([a, b]) == isd.DoSHistogram(spec, table)
    assert isd.merge([], spec=spec).total() == 0
    with pytest.raises(ValueError):
        isd.merge([])
    with pytest.raises(ValueError):
        a + isd.DoSHistogram(isd.LatticeSpec(3, 3, coupling=-1))
    with pytest.raises(ValueError):
        isd.merge([a], spec=isd.LatticeSpec(3, 3, coupling=-1))


def test_verify_flags_each_perturbation():
    rows, cols, depth, j, table = read_csv_table("dos_4x4x1_J1.csv")
    spec = isd.LatticeSpec(rows, cols, depth, j)
    good = isd.verify_dos(isd.DoSHistogram(spec, table))
    assert good.passed and len(good.checks) == 4
    t = table.copy()
    t[8, 16] += 1  # one extra count in (M=0, E=0)
    rep = isd.verify_dos(isd.DoSHistogram(spec, t))
    assert set(rep.failed_names()) == {"total-count", "binomial-marginals"}
    t = table.copy()
    t[9, 16] += 1
    t[9, 14] -= 1  # moves a count: marginals hold, flip symmetry breaks
    rep = isd.verify_dos(isd.DoSHistogram(spec, t))
    assert rep.failed_names() == ["flip-symmetry"]


# -- tables and thermodynamics on the GPU ---------------------------------------

def _dos(name):
    rows, cols, depth, j, table = read_csv_table(name)
    return isd.DoSHistogram(isd.LatticeSpec(rows, cols, depth, j), table)


@pytest.mark.gpu
def test_antiferromagnet_mirrors_ferromagnet():
    # J -> -J maps E -> -E: g_{-J}(M, E) = g_J(M, -E)  (test_enumeration.py:214-219)
    for dims in ((4, 4), (3, 4), (2, 2, 2)):
        f = isd.full_dos(isd.LatticeSpec(*dims))
        a = isd.full_dos(isd.LatticeSpec(*dims, coupling=-1))
        assert np.array_equal(a.counts, f.counts[:, ::-1])


@pytest.mark.gpu
def test_batch_size_and_shard_count_invisible():
    spec = isd.LatticeSpec(3, 4)
    whole = isd.enumerate_shard(spec, None, isd.make_shards(spec, 1)[0])
    for bs in (1, 7, 8192, 1 << 20):
        assert isd.enumerate_shard(spec, None, isd.make_shards(spec, 1)[0],
                                   batch_size=bs) == whole
    for p in (2, 3, 5, 7, 16):
        parts = [isd.enumerate_shard(spec, None, s)
                 for s in isd.make_shards(spec, p)]
        assert all(pt.total() == s.size
                   for pt, s in zip(parts, isd.make_shards(spec, p)))
        assert isd.merge(parts) == whole
    with pytest.raises(ValueError):
        isd.enumerate_shard(spec, None, isd.make_shards(spec, 1)[0],
                            batch_size=0)


@pytest.mark.gpu
def test_thermo_limits_and_identities():
    dos = _dos("dos_4x4x1_J1.csv")
    n = 16
    hot = isd.partition_point(dos, 0.0, 1e6)  # T -> inf: Z -> 2^N
    assert abs(hot.log_z - n * math.log(2)) < 1e-3
    cold = isd.partition_point(dos, 0.0, 0.05)  # T -> 0: two ground states
    assert abs(cold.internal_energy + 32) < 1e-9
    assert abs(cold.log_z - (32 / 0.05 + math.log(2))) < 1e-9
    for t in (0.7, 2.3, 4.0):
        p = isd.partition_point(dos, 0.0, t)
        assert p.free_energy == -t * p.log_z
        assert abs(p.mean_magnetization) < 1e-12
        assert p.specific_heat >= 0 and p.susceptibility >= 0
        assert 0 < p.mean_abs_magnetization <= n
        up = isd.partition_point(dos, 0.3, t)
        down = isd.partition_point(dos, -0.3, t)
        assert abs(up.mean_magnetization + down.mean_magnetization) < 1e-12
        assert abs(up.log_z - down.log_z) < 1e-12
        # log Z >= the ground-state term, <= N log 2 + max(-E/T)
        assert p.log_z >= 32 / t and p.log_z <= n * math.log(2) + 32 / t


@pytest.mark.gpu
def test_specific_heat_has_one_peak():
    dos = _dos("dos_5x5x1_J1.csv")
    temps = [0.5 + 0.01 * i for i in range(451)]
    c = [p.specific_heat for p in isd.thermo_sweep(dos, 0.0, temps)]
    peak = int(np.argmax(c))
    assert 0 < peak < len(c) - 1
    assert all(c[i] <= c[i + 1] + 1e-12 for i in range(peak - 5))
    assert all(c[i] >= c[i + 1] - 1e-12 for i in range(peak + 5, len(c) - 1))


# -- cross-check API (the reference's oracle.py names) ----------------------

def test_crosscheck_scalar_helpers_match_naive_oracle():
    from oracle import naive
    rng = random.Random(5)
    for dims, kw in [((3, 4, 1), {}), ((2, 2, 3), {}), ((2, 3, 1), {}),
                     ((4, 4, 1), dict(boundary="free")), ((3, 3, 2), {})]:
        for j in (1, -2.5, 0.5):
            spec = isd.LatticeSpec(*dims, j, **kw)
            assert len(isd.crosscheck.bond_pairs(spec)) == spec.num_bonds
            for x in rng.sample(range(spec.num_configs), 40):
                spins = isd.decode_spins(spec, x)
                assert len(spins) == spec.num_spins
                assert isd.oracle_energy(spins, spec) == naive.energy_of(
                    *dims, x, j, spec.periodic)
                assert isd.oracle_energy(spins, spec) == isd.total_energy(
                    isd.decode_config(spec, x), spec)
                assert isd.oracle_magnetization(spins) == isd.spin_excess(
                    isd.decode_config(spec, x), spec)


def test_crosscheck_signed_energy_matches_unsatisfied_bonds():
    base = isd.LatticeSpec(3, 4)
    spec = isd.LatticeSpec(3, 4, bond_signs=isd.random_bond_signs(base, 9))
    for x in range(0, spec.num_configs, 97):
        e_idx = isd.unsatisfied_bonds(spec, x)
        assert isd.oracle_energy(isd.decode_spins(spec, x), spec) == \
            2 * e_idx - spec.num_bonds


def test_crosscheck_caps_and_validation():
    big = isd.LatticeSpec(5, 5)
    with pytest.raises(ValueError, match="oracle cap of 24"):
        isd.oracle_full_dos(big)
    with pytest.raises(ValueError, match="oracle cap"):
        isd.brute_force_log_z(big, 0.0, 1.0)
    with pytest.raises(ValueError, match="temperature"):
        isd.brute_force_log_z(isd.LatticeSpec(2, 2), 0.0, 0.0)
    with pytest.raises(ValueError):
        isd.decode_spins(isd.LatticeSpec(2, 2), 16)
    assert isd.ORACLE_MAX_SPINS == 24


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dos_2x2x1_J1.csv", "dos_3x3x1_J1.csv",
                                  "dos_4x4x1_J1.csv", "dos_2x2x2_J1.csv"])
def test_crosscheck_route_reproduces_reference_tables(name):
    rows, cols, depth, j, table = read_csv_table(name)
    spec = isd.LatticeSpec(rows, cols, depth, j)
    got = isd.oracle_full_dos(spec)
    assert np.array_equal(got.counts, table)
    assert got == isd.full_dos(spec)


@pytest.mark.gpu
def test_brute_force_log_z_matches_partition_point():
    for dims, kw in [((4, 4), {}), ((3, 4), dict(coupling=-1)),
                     ((4, 4), dict(boundary="free"))]:
        spec = isd.LatticeSpec(*dims, **kw)
        dos = isd.full_dos(spec)
        for h, t in ((0.0, 1.0), (0.3, 2.5), (-0.2, 4.0)):
            bf = isd.brute_force_log_z(spec, h, t)
            lz = isd.partition_point(dos, h, t).log_z
            assert abs(bf - lz) <= 1e-12 * abs(lz)


@pytest.mark.gpu
def test_cli_oracle_check(capsys):
    from paper_1110_2561_b200.cli import main
    assert main(["oracle-check", "--rows", "3", "--cols", "4"]) == 0
    assert "OK: bit-kernel and naive engines agree on all 4096" in \
        capsys.readouterr().out
    assert main(["oracle-check", "--rows", "5", "--cols", "5"]) == 1
    assert "oracle cap" in capsys.readouterr().err


# -- independence of the shipped cross-check ------------------

def test_crosscheck_bond_pairs_restate_geometry_in_reference_order():
    # crosscheck.bond_pairs walks the lattice itself (oracle.py:40-58); the
    # order is the contract bond_signs is defined in, so it must equal the
    # order of LatticeSpec.bond_list() without being computed from it
    for dims in [(2, 2, 1), (3, 3, 1), (4, 4, 1), (2, 3, 2), (3, 3, 4),
                 (2, 2, 2), (4, 3, 3), (2, 5, 4), (6, 6, 1)]:
        for bd in ("periodic", "free"):
            spec = isd.LatticeSpec(*dims, boundary=bd)
            slot = {spec.bit_position(r, c, l): i for i, (r, c, l)
                    in enumerate(isd.crosscheck.site_order(spec))}
            want = [(slot[i], slot[j]) for i, j, _, _ in spec.bond_list()]
            assert isd.crosscheck.bond_pairs(spec) == want


def test_crosscheck_never_consults_the_bond_classes(monkeypatch):
    # the naive route must not read the descriptor K1 runs on: break every
    # route to it and capture what reaches the naive engine
    from paper_1110_2561_b200 import _native
    from oracle import naive
    seen = {}

    def capture(bits, bonds, sign, start, end, device=None):
        seen.update(bits=bits, bonds=bonds, sign=sign, range=(start, end))
        return np.zeros((spec.num_spins + 1, spec.num_bonds + 1),
                        dtype=np.uint64)

    def boom(*a, **k):
        raise AssertionError("the cross-check touched the fast path")

    monkeypatch.setattr(isd.LatticeSpec, "bond_classes", boom)
    monkeypatch.setattr(isd.LatticeSpec, "bond_list", boom)
    monkeypatch.setattr(_native, "naive_enumerate", capture)
    monkeypatch.setattr(_native, "enumerate_host", boom)
    base = isd.LatticeSpec(3, 4, 2)
    signs = naive.random_signs(base.num_bonds, 11)
    spec = isd.LatticeSpec(3, 4, 2, -1.5, bond_signs=signs)
    isd.oracle_full_dos(spec)
    assert seen["sign"] == -1 and seen["range"] == (0, spec.num_configs)
    assert sorted(seen["bits"]) == list(range(spec.num_spins))
    assert len(seen["bonds"]) == spec.num_bonds
    # the bond list agrees with the test oracle's per-bond restatement
    pairs = naive.bond_pairs(3, 4, 2, True)
    assert [(i, j) for i, j, _ in seen["bonds"]] == [tuple(p) for p in pairs]


@pytest.mark.gpu
def test_oracle_check_catches_a_fault_in_the_bond_classes(monkeypatch, capsys):
    # inject a fault into the descriptor the fast path compiles (one bond's
    # sign flipped in its class masks): the naive engine must disagree
    from paper_1110_2561_b200 import enumeration
    from paper_1110_2561_b200.cli import main
    good = isd.LatticeSpec.bond_classes

    def faulty(self):
        classes = list(good(self))
        s, m, j = classes[0]
        low = m & -m
        classes[0] = (s, m, j ^ low)
        return classes

    monkeypatch.setattr(isd.LatticeSpec, "bond_classes", faulty)
    monkeypatch.setattr(enumeration, "_DESCRIPTORS", {})
    assert main(["oracle-check", "--rows", "3", "--cols", "4"]) == 1
    assert "mismatching cells" in capsys.readouterr().err
    monkeypatch.setattr(isd.LatticeSpec, "bond_classes", good)
    monkeypatch.setattr(enumeration, "_DESCRIPTORS", {})
    assert main(["oracle-check", "--rows", "3", "--cols", "4"]) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("kw", [dict(boundary="free"), dict(coupling=-2),
                                dict(seed=3)])
def test_naive_engine_matches_fast_path_on_extended_lattices(kw):
    kw = dict(kw)
    seed = kw.pop("seed", None)
    base = isd.LatticeSpec(3, 4, 2, **kw)
    spec = base if seed is None else isd.LatticeSpec(
        3, 4, 2, bond_signs=isd.random_bond_signs(base, seed))
    got = isd.oracle_full_dos(spec)
    assert got == isd.full_dos(spec)
    assert isd.verify_dos(got).passed
