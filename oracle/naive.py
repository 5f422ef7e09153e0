"""Naive oracle: explicit spin arrays and per-bond loops (TEST ONLY).

Restates /root/reference/pkg/src/isingdos/oracle.py with two extensions the
reference lacks: free boundaries (wrap bonds dropped) and per-bond signs.
Deliberately shares no code with paper_1110_2561_b200 (own site order, own
bond list, own bit positions), so agreement is evidence, not tautology.
"""

import math

import numpy as np

#: oracle.py:16
ORACLE_MAX_SPINS = 24


def site_order(rows, cols, depth):
    """(row, col, layer) triples, row-major (oracle.py:19-24)."""
    return [(r, c, l) for r in range(rows) for c in range(cols)
            for l in range(depth)]


def bit_position(rows, cols, r, c, l):
    """oracle.py:27-29."""
    return (l * cols + c) * rows + r


def bond_pairs(rows, cols, depth, periodic=True):
    """Spin-array index pairs, one per bond (oracle.py:40-58).

    Each site pairs with its +1 neighbour along rows, cols and (depth > 1)
    layers; free boundaries skip the neighbour that would wrap.
    """
    flat = {rcl: i for i, rcl in enumerate(site_order(rows, cols, depth))}
    dims = (rows, cols, depth)
    pairs = []
    for r, c, l in site_order(rows, cols, depth):
        here = flat[(r, c, l)]
        axes = 3 if depth > 1 else 2
        for a in range(axes):
            coord = (r, c, l)
            if not periodic and coord[a] + 1 >= dims[a]:
                continue
            nxt = list(coord)
            nxt[a] = (nxt[a] + 1) % dims[a]
            pairs.append((here, flat[tuple(nxt)]))
    return pairs


def random_signs(n_bonds, seed, p_plus=0.5):
    """The frozen BASELINE config-4 convention."""
    draws = np.random.default_rng(seed).random(n_bonds)
    return [1 if x < p_plus else -1 for x in draws]


def full_dos(rows, cols, depth=1, coupling=1, periodic=True, signs=None):
    """Exact g(M, E) as an int64 (N+1, B+1) array (oracle.py:71-91).

    e_idx = (E/|J| + B)/2 with E = -sum_b J_b s_i s_j, J_b = coupling*sign_b.
    """
    n = rows * cols * depth
    if n > ORACLE_MAX_SPINS:
        raise ValueError(f"{n} spins exceeds the oracle cap of {ORACLE_MAX_SPINS}")
    positions = [bit_position(rows, cols, r, c, l)
                 for r, c, l in site_order(rows, cols, depth)]
    pairs = bond_pairs(rows, cols, depth, periodic)
    b = len(pairs)
    signs = signs or [1] * b
    jb = [coupling * s for s in signs]
    scale = abs(coupling)
    counts = np.zeros((n + 1, b + 1), dtype=np.int64)
    for index in range(1 << n):
        spins = [1 if (index >> p) & 1 else -1 for p in positions]
        m = sum(spins)
        e = -sum(j * spins[i] * spins[k] for (i, k), j in zip(pairs, jb))
        unit = e / scale
        iu = int(round(unit))
        assert abs(unit - iu) < 1e-9
        counts[(m + n) // 2, (iu + b) // 2] += 1
    return counts


def energy_of(rows, cols, depth, index, coupling=1, periodic=True, signs=None):
    """E of one configuration index, per-bond (oracle.py:61-63)."""
    positions = [bit_position(rows, cols, r, c, l)
                 for r, c, l in site_order(rows, cols, depth)]
    spins = [1 if (index >> p) & 1 else -1 for p in positions]
    pairs = bond_pairs(rows, cols, depth, periodic)
    signs = signs or [1] * len(pairs)
    return -sum(coupling * s * spins[i] * spins[k]
                for (i, k), s in zip(pairs, signs))


def brute_force_log_z(rows, cols, depth, h, temperature, coupling=1,
                      periodic=True, signs=None):
    """log Z by direct fsum of exp(-(E - hM)/T) (oracle.py:94-116)."""
    n = rows * cols * depth
    if n > ORACLE_MAX_SPINS:
        raise ValueError(f"{n} spins exceeds the oracle cap of {ORACLE_MAX_SPINS}")
    positions = [bit_position(rows, cols, r, c, l)
                 for r, c, l in site_order(rows, cols, depth)]
    pairs = bond_pairs(rows, cols, depth, periodic)
    signs = signs or [1] * len(pairs)
    terms = []
    for index in range(1 << n):
        spins = [1 if (index >> p) & 1 else -1 for p in positions]
        m = sum(spins)
        e = -sum(coupling * s * spins[i] * spins[k]
                 for (i, k), s in zip(pairs, signs))
        terms.append(math.exp(-(e - h * m) / temperature))
    return math.log(math.fsum(terms))
