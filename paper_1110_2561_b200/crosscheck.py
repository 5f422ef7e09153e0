"""The reference's cross-check API (oracle.py:1-116), backed by a second
GPU formulation.

The reference ships a deliberately naive engine next to its fast one so
that agreement between the two is evidence rather than tautology.  The same
names live here with the same signatures, caps and messages, but the
"naive" side is the canonical kernel K1a: one thread per configuration
evaluating every bond class from scratch (`ALGO_CANONICAL`), which shares
no code path with the hoisted kernel beyond the bond-class descriptor.
There is no CPU walk: like every compute call in this package these raise
without a GPU.  The per-configuration helpers (`decode_spins`,
`oracle_energy`, `oracle_magnetization`) are host-side scalar definitions,
as in the reference.

The 24-spin cap is kept for drop-in behaviour (the reference's tests and
CLI rely on its message); the GPU route itself has no such limit.
"""

import math

import numpy as np

from . import _native
from .enumeration import DoSHistogram, enumerate_range_timed
from .lattice import LatticeSpec

#: oracle.py:18 — the reference's cap on the naive walk.
ORACLE_MAX_SPINS = 24


def site_order(spec: LatticeSpec) -> list[tuple[int, int, int]]:
    """(row, col, layer) of each spin-array slot, row-major (oracle.py:19-24)."""
    return [(r, c, l) for r in range(spec.rows) for c in range(spec.cols)
            for l in range(spec.depth)]


def _slot_of_bit(spec: LatticeSpec) -> dict:
    return {spec.bit_position(r, c, l): i
            for i, (r, c, l) in enumerate(site_order(spec))}


def decode_spins(spec: LatticeSpec, index: int) -> list[int]:
    """+1 / -1 per site in `site_order` (oracle.py:32-37)."""
    if not 0 <= index < spec.num_configs:
        raise ValueError(f"index {index} outside [0, 2^{spec.num_spins})")
    return [2 * ((index >> spec.bit_position(r, c, l)) & 1) - 1
            for r, c, l in site_order(spec)]


def bond_pairs(spec: LatticeSpec) -> list[tuple[int, int]]:
    """Every bond once as a pair of spin-array slots (oracle.py:40-58).

    Reference order; a periodic axis of length 2 lists its two bonds, free
    boundaries (an extension) leave out the wrap bonds.
    """
    slot = _slot_of_bit(spec)
    return [(slot[i], slot[j]) for i, j, _, _ in spec.bond_list()]


def oracle_energy(spins, spec: LatticeSpec):
    """E = -J * sum over bonds of sign_b S_i S_j (oracle.py:61-63)."""
    slot = _slot_of_bit(spec)
    total = sum(sign * spins[slot[i]] * spins[slot[j]]
                for i, j, _, sign in spec.bond_list())
    return -spec.coupling * total


def oracle_magnetization(spins) -> int:
    """M = sum of the spin values (oracle.py:66-68)."""
    return sum(spins)


def _check_cap(spec: LatticeSpec) -> None:
    n = spec.num_spins
    if n > ORACLE_MAX_SPINS:
        raise ValueError(
            f"{n} spins exceeds the oracle cap of {ORACLE_MAX_SPINS}")


def _canonical_counts(spec: LatticeSpec) -> np.ndarray:
    table, _ = enumerate_range_timed(spec, 0, spec.num_configs,
                                     algo=_native.ALGO_CANONICAL)
    return table.view(np.int64)


def oracle_full_dos(spec: LatticeSpec) -> DoSHistogram:
    """g(M, E) of all 2^N configurations through the canonical kernel.

    Raises ValueError over the cap (oracle.py:71-91).
    """
    _check_cap(spec)
    return DoSHistogram(spec, _canonical_counts(spec))


def brute_force_log_z(spec: LatticeSpec, h: float, temperature: float) -> float:
    """log Z by plain summation of exp(-H/T), no log-sum-exp shift
    (oracle.py:94-116).

    The canonical kernel's table groups the 2^N Boltzmann terms by (M, E);
    each group contributes g * exp(-(E - hM)/T), summed with fsum.
    """
    if temperature <= 0:
        raise ValueError(f"temperature must be > 0, got {temperature}")
    _check_cap(spec)
    dos = DoSHistogram(spec, _canonical_counts(spec))
    terms = [count * math.exp(-(e - h * m) / temperature)
             for count, m, e in dos.cells()]
    return math.log(math.fsum(terms))
