"""The reference's cross-check API (oracle.py:1-116), backed by a naive GPU
engine that shares nothing with the fast path.

The reference ships a deliberately naive engine next to its fast one so
that agreement between the two is evidence rather than tautology
(separate decode, separate neighbour enumeration).  The same
names live here with the same signatures, caps and messages.  Everything
below is built from the lattice geometry alone, restating oracle.py: the
site order, the bit of each site, and every bond as a pair of spin-array
slots walked site by site (+row, +col, +layer neighbour).  It never touches
`LatticeSpec.bond_classes()` / `bond_list()`, the bond-class descriptor,
or the enumeration kernels: configurations are counted by K5
(`isd_naive_enumerate`, csrc/naive.cu), one thread per configuration
decoding every spin and summing S_i S_j over the explicit bond list.  A
fault in the bond classes or in K1 therefore makes `oracle-check` fail.
There is no CPU walk: like every compute call in this package these raise
without a GPU.  `decode_spins`, `oracle_energy` and `oracle_magnetization`
are host-side scalar definitions, as in the reference.

The 24-spin cap is kept for drop-in behaviour (the reference's tests and
CLI rely on its message); the GPU route itself has no such limit.
"""

import math

from . import _native
from .enumeration import DoSHistogram
from .lattice import LatticeSpec

#: oracle.py:18 — the reference's cap on the naive walk.
ORACLE_MAX_SPINS = 24


def site_order(spec: LatticeSpec) -> list[tuple[int, int, int]]:
    """(row, col, layer) of each spin-array slot, row-major (oracle.py:19-24)."""
    return [(r, c, l) for r in range(spec.rows) for c in range(spec.cols)
            for l in range(spec.depth)]


def _bit_position(spec: LatticeSpec, r: int, c: int, l: int) -> int:
    """Index bit of site (r, c, l) (oracle.py:27-29)."""
    return (l * spec.cols + c) * spec.rows + r


def decode_spins(spec: LatticeSpec, index: int) -> list[int]:
    """+1 / -1 per site in `site_order` (oracle.py:32-37)."""
    if not 0 <= index < spec.num_configs:
        raise ValueError(f"index {index} outside [0, 2^{spec.num_spins})")
    return [1 if (index >> _bit_position(spec, r, c, l)) & 1 else -1
            for r, c, l in site_order(spec)]


def bond_pairs(spec: LatticeSpec) -> list[tuple[int, int]]:
    """Every bond once as a pair of spin-array slots (oracle.py:40-58).

    Each site is paired with its +1 neighbour along every axis (rows, cols,
    and layers when depth > 1), so a periodic axis of length 2 contributes
    the same two sites twice (its two bonds).  With free boundaries (an
    extension) the pair across the edge is left out.
    """
    flat = {rcl: i for i, rcl in enumerate(site_order(spec))}
    dims = (spec.rows, spec.cols, spec.depth)
    pairs = []
    for r, c, l in site_order(spec):
        here = flat[(r, c, l)]
        for axis in range(3 if spec.depth > 1 else 2):
            coord = (r, c, l)[axis]
            if not spec.periodic and coord + 1 == dims[axis]:
                continue
            nxt = [r, c, l]
            nxt[axis] = (coord + 1) % dims[axis]
            pairs.append((here, flat[tuple(nxt)]))
    return pairs


def _bond_signs(spec: LatticeSpec) -> list[int]:
    """Per-bond signs in bond_pairs order (the order `bond_signs` is
    defined in; +1 everywhere for a uniform lattice)."""
    n = len(bond_pairs(spec))
    signs = list(spec.bond_signs) if spec.bond_signs else [1] * n
    if len(signs) != n:
        raise ValueError(f"{len(signs)} bond signs for {n} bonds")
    return signs


def oracle_energy(spins, spec: LatticeSpec):
    """E = -J * sum over bonds of sign_b S_i S_j (oracle.py:61-63)."""
    return -spec.coupling * sum(
        sign * spins[i] * spins[j]
        for (i, j), sign in zip(bond_pairs(spec), _bond_signs(spec)))


def oracle_magnetization(spins) -> int:
    """M = sum of the spin values (oracle.py:66-68)."""
    return sum(spins)


def _check_cap(spec: LatticeSpec) -> None:
    n = spec.num_spins
    if n > ORACLE_MAX_SPINS:
        raise ValueError(
            f"{n} spins exceeds the oracle cap of {ORACLE_MAX_SPINS}")


def _naive_counts(spec: LatticeSpec):
    """int64 g(M, E) of all 2^N configurations from the naive engine K5."""
    bits = [_bit_position(spec, r, c, l) for r, c, l in site_order(spec)]
    bonds = [(i, j, sign) for (i, j), sign
             in zip(bond_pairs(spec), _bond_signs(spec))]
    table = _native.naive_enumerate(bits, bonds, 1 if spec.coupling > 0 else -1,
                                    0, spec.num_configs)
    return table.view("int64")


def oracle_full_dos(spec: LatticeSpec) -> DoSHistogram:
    """g(M, E) of all 2^N configurations through the naive engine.

    Raises ValueError over the cap (oracle.py:71-91).
    """
    _check_cap(spec)
    return DoSHistogram(spec, _naive_counts(spec))


def brute_force_log_z(spec: LatticeSpec, h: float, temperature: float) -> float:
    """log Z by plain summation of exp(-H/T), no log-sum-exp shift
    (oracle.py:94-116).

    The naive engine's table groups the 2^N Boltzmann terms by (M, E);
    each group contributes g * exp(-(E - hM)/T), summed with fsum.
    """
    if temperature <= 0:
        raise ValueError(f"temperature must be > 0, got {temperature}")
    _check_cap(spec)
    dos = DoSHistogram(spec, _naive_counts(spec))
    terms = [count * math.exp(-(e - h * m) / temperature)
             for count, m, e in dos.cells()]
    return math.log(math.fsum(terms))
