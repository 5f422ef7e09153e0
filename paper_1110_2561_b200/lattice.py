"""Lattice geometry, bit layout and the bond-class compiler.

Mirrors the reference module /root/reference/pkg/src/isingdos/lattice.py:
the same `LatticeSpec(rows, cols, depth=1, coupling=1)` value type with the
same validation messages (lattice.py:50-75), the same index layout
(bit of site (row, col, layer) = (layer*cols + col)*rows + row,
lattice.py:1-13 and oracle.py:27-29) and the same scalar per-configuration
helpers (lattice.py:130-261).

Two keyword-only extensions (BASELINE configs 1, 3 and 4 need them; the
reference expresses only periodic, uniform-J lattices, lattice.py:83-85):

* ``boundary="free"`` drops the wrap-around bonds of every axis;
* ``bond_signs=(+1, -1, ...)`` gives one sign per bond, in the reference's
  bond order (oracle.bond_pairs, oracle.py:40-58: sites row-major over
  (row, col, layer); per site its +row, +col and, in 3D, +layer bond; free
  boundaries skip the wrap bonds).  J_ij = coupling * sign.

Defaults reproduce the reference exactly, including positional
construction, frozen-dataclass equality and `num_bonds`.

The GPU engine sees a lattice only as bond classes (`bond_classes`): per
axis an "interior" class (partner at +stride) and, if periodic, a "wrap"
class (partner at +(L-1)*stride), each a (shift, bond_mask, jneg_mask)
triple over the N-bit index.  A periodic axis of length 2 yields two
classes with the same pairs: the reference's double bond
(lattice.py:105-107, oracle.py:43-46).
"""

from dataclasses import dataclass, field

import numpy as np

#: lattice.py:24 — the configuration index must fit a 64-bit word.
MAX_SPINS = 40
#: lattice.py:27 — a column word fits a 32-bit significant-bit mask.
MAX_ROWS = 30
#: lattice.py:31 — lookup tables exist up to 2^16 entries.
TABLE_ROWS_CAP = 16

BOUNDARIES = ("periodic", "free")


def _check_geometry(rows, cols, depth) -> None:
    """The reference's geometry rules and messages (lattice.py:50-70)."""
    for label, value in (("rows", rows), ("cols", cols), ("depth", depth)):
        if isinstance(value, bool) or not isinstance(value, int):
            raise ValueError(f"{label} must be an integer, got {value!r}")
    if min(rows, cols) < 2:
        raise ValueError("degenerate periodic axis: rows and cols must be "
                         f">= 2, got rows={rows} cols={cols}")
    if depth < 1:
        raise ValueError(f"depth must be >= 1, got {depth}")
    if rows > MAX_ROWS:
        raise ValueError(f"rows={rows} exceeds the cap of {MAX_ROWS}")
    spins = rows * cols * depth
    if spins > MAX_SPINS:
        raise ValueError(f"{spins} spins exceeds the cap of {MAX_SPINS} "
                         "(2^N must fit a 64-bit index with headroom)")


def _check_signs(signs, n_bonds: int) -> tuple:
    signs = tuple(signs)
    if len(signs) != n_bonds:
        raise ValueError(f"bond_signs has {len(signs)} entries, lattice has "
                         f"{n_bonds} bonds")
    bad = next((x for x in signs if isinstance(x, bool) or x not in (1, -1)),
               None)
    if bad is not None:
        raise ValueError(f"bond signs must be +1 or -1, got {bad!r}")
    return tuple(int(x) for x in signs)


@dataclass(frozen=True)
class LatticeSpec:
    """Geometry and couplings of a finite Ising lattice.

    rows:       column height n (spins per bit-word), 2..30
    cols:       number of columns, >= 2
    depth:      number of layers; 1 for 2D, >= 2 for 3D
    coupling:   exchange constant J (nonzero; integral floats become ints)
    boundary:   "periodic" (reference behaviour) or "free"
    bond_signs: None (uniform J) or one +1/-1 per bond in bond_list() order
    """

    rows: int
    cols: int
    depth: int = 1
    coupling: float = 1
    boundary: str = field(default="periodic", kw_only=True)
    bond_signs: tuple | None = field(default=None, kw_only=True)

    def __post_init__(self):
        _check_geometry(self.rows, self.cols, self.depth)
        j = self.coupling
        if j == 0:
            raise ValueError("coupling J must be nonzero")
        if isinstance(j, float) and j.is_integer():
            # integral J stays an int so energies remain exact integers
            object.__setattr__(self, "coupling", int(j))
        if self.boundary not in BOUNDARIES:
            raise ValueError(
                f"boundary must be one of {BOUNDARIES}, got {self.boundary!r}")
        if self.bond_signs is not None:
            object.__setattr__(self, "bond_signs",
                               _check_signs(self.bond_signs, self.num_bonds))

    # -- derived sizes (lattice.py:77-100) ---------------------------------

    @property
    def num_spins(self) -> int:
        return self.rows * self.cols * self.depth

    @property
    def periodic(self) -> bool:
        return self.boundary == "periodic"

    @property
    def num_bonds(self) -> int:
        """Bond count B: 2N (2D) / 3N (3D) periodic, fewer with free edges."""
        r, c, d = self.rows, self.cols, self.depth
        if self.periodic:
            return (2 if d == 1 else 3) * self.num_spins
        return (r - 1) * c * d + r * (c - 1) * d + r * c * (d - 1)

    @property
    def num_words(self) -> int:
        return self.cols * self.depth

    @property
    def num_configs(self) -> int:
        return 1 << self.num_spins

    @property
    def word_mask(self) -> int:
        return (1 << self.rows) - 1

    @property
    def uniform(self) -> bool:
        """True for the reference's lattices: periodic with one scalar J."""
        return self.periodic and self.bond_signs is None

    def word_neighbor_pairs(self) -> list[tuple[int, int]]:
        """Inter-word bond pairs: the col axis, then (3D) the layer axis.

        Order of lattice.py:102-119; free boundaries leave out the wrap
        pairs, and a periodic axis of length 2 lists both orders of the
        same two words (its double bond).
        """
        cols, depth = self.cols, self.depth

        def word(c, layer):
            return layer * cols + c

        col_pairs = [(word(c, layer), word((c + 1) % cols, layer))
                     for layer in range(depth) for c in range(cols)
                     if self.periodic or c < cols - 1]
        if depth == 1:
            return col_pairs
        layer_pairs = [(word(c, layer), word(c, (layer + 1) % depth))
                       for layer in range(depth) for c in range(cols)
                       if self.periodic or layer < depth - 1]
        return col_pairs + layer_pairs

    # -- bond geometry ------------------------------------------------------

    def bit_position(self, r: int, c: int, l: int = 0) -> int:
        """Index bit of site (row, col, layer) (oracle.py:27-29)."""
        return (l * self.cols + c) * self.rows + r

    def _bonds(self) -> list[tuple[int, int, int, bool]]:
        """(bit_here, bit_next, axis, wraps) in the reference bond order."""
        dims = (self.rows, self.cols, self.depth)
        axes = 3 if self.depth > 1 else 2
        out = []
        for r in range(self.rows):
            for c in range(self.cols):
                for l in range(self.depth):
                    here = (r, c, l)
                    for a in range(axes):
                        wraps = here[a] + 1 >= dims[a]
                        if wraps and not self.periodic:
                            continue
                        nxt = list(here)
                        nxt[a] = (nxt[a] + 1) % dims[a]
                        out.append((self.bit_position(*here),
                                    self.bit_position(*nxt), a, wraps))
        return out

    def bond_list(self) -> list[tuple[int, int, int, int]]:
        """Every bond once as (bit_i, bit_j, axis, sign), reference order.

        Order follows oracle.bond_pairs (oracle.py:40-58): sites row-major
        over (row, col, layer); per site the +row, +col and (3D) +layer
        neighbour.  axis 0/1/2 = rows/cols/layers.  sign is the bond's
        entry of bond_signs (+1 when uniform).
        """
        bonds = self._bonds()
        signs = self.bond_signs or (1,) * len(bonds)
        return [(i, j, a, s) for (i, j, a, _), s in zip(bonds, signs)]

    def bond_classes(self) -> list[tuple[int, int, int]]:
        """Compile the bonds into (shift, bond_mask, jneg_mask) classes.

        Interior bond of axis a: lower site = here, partner at +stride_a.
        Wrap bond (periodic only): lower site = the neighbour at coordinate
        0, partner at +(L_a - 1) * stride_a.  jneg marks bonds whose
        effective sign sign(J) * bond_sign is negative (unsatisfied when
        aligned).  Classes come out ordered (axis, interior, wrap).
        """
        dims = (self.rows, self.cols, self.depth)
        strides = (1, self.rows, self.rows * self.cols)
        neg_j = self.coupling < 0
        signs = self.bond_signs or (1,) * self.num_bonds
        masks = {}
        for (i, j, a, wraps), s in zip(self._bonds(), signs):
            if wraps:
                lo, shift = j, (dims[a] - 1) * strides[a]
            else:
                lo, shift = i, strides[a]
            m, jn, _ = masks.get((a, wraps), (0, 0, shift))
            m |= 1 << lo
            if (s < 0) != neg_j:
                jn |= 1 << lo
            masks[(a, wraps)] = (m, jn, shift)
        out = []
        for a in range(3):
            for wraps in (False, True):
                if (a, wraps) in masks:
                    m, jn, shift = masks[(a, wraps)]
                    out.append((shift, m, jn))
        return out


@dataclass(frozen=True)
class Configuration:
    """One spin configuration: its global index and decoded column words."""

    index: int
    words: tuple[int, ...]


def decode_config(spec: LatticeSpec, index: int) -> Configuration:
    """Split an index into its column bit-words (lattice.py:130-137)."""
    if index < 0 or index >= spec.num_configs:
        raise ValueError(f"index {index} outside [0, 2^{spec.num_spins})")
    h, mask = spec.rows, spec.word_mask
    return Configuration(index, tuple((index >> shift) & mask for shift
                                      in range(0, h * spec.num_words, h)))


def encode_words(spec: LatticeSpec, words) -> int:
    """Inverse of decode_config (lattice.py:140-148)."""
    if len(words) != spec.num_words:
        raise ValueError(f"expected {spec.num_words} words, got {len(words)}")
    packed = 0
    for word in reversed(words):
        if word < 0 or word > spec.word_mask:
            raise ValueError(
                f"word {word:#x} has stray bits above row {spec.rows}")
        packed = (packed << spec.rows) | word
    return packed


@dataclass(frozen=True, eq=False)
class KernelTables:
    """Per-word popcount / circular-shift tables (lattice.py:151-164).

    Kept for API compatibility: `enumerate_shard` accepts and ignores them,
    because the GPU kernels use hardware POPC and funnel shifts instead.
    """

    rows: int
    mask: int
    popcount_table: np.ndarray = field(repr=False)
    shift_table: np.ndarray = field(repr=False)


def build_tables(rows: int) -> KernelTables:
    """popcount and circular-left-shift tables of length 2^rows."""
    if not 2 <= rows <= TABLE_ROWS_CAP:
        raise ValueError(
            f"tables support 2 <= rows <= {TABLE_ROWS_CAP}, got {rows}")
    size = 1 << rows
    j = np.arange(size, dtype=np.int64)
    pc = np.bitwise_count(j.astype(np.uint64)).astype(np.int64)
    shift = ((j << 1) | (j >> (rows - 1))) & (size - 1)
    return KernelTables(rows=rows, mask=size - 1, popcount_table=pc,
                        shift_table=shift)


def popcount(word: int) -> int:
    """Number of set bits of a nonnegative integer."""
    return int(word).bit_count()


def circular_shift(word: int, rows: int) -> int:
    """Circular left shift of the rows significant bits of word by one."""
    mask = (1 << rows) - 1
    return ((word << 1) | (word >> (rows - 1))) & mask


def spin_excess(config: Configuration, spec: LatticeSpec) -> int:
    """M = 2 * (#up) - N (lattice.py:200-207)."""
    return 2 * sum(popcount(w) for w in config.words) - spec.num_spins


def aligned_row_bonds(word_a: int, word_b: int, tables: KernelTables) -> int:
    """Aligned bonds between neighbouring columns (lattice.py:210-217)."""
    return int(tables.popcount_table[(word_a ^ word_b) ^ tables.mask])


def aligned_column_bonds(word: int, tables: KernelTables) -> int:
    """Aligned periodic vertical pairs in one column (lattice.py:220-227)."""
    shifted = int(tables.shift_table[word])
    return int(tables.popcount_table[(word ^ shifted) ^ tables.mask])


def unsatisfied_bonds(spec: LatticeSpec, index: int) -> int:
    """e_idx of one configuration via the bond classes (the K1 contract)."""
    e = 0
    for s, m, jn in spec.bond_classes():
        e += popcount(((index ^ (index >> s)) ^ jn) & m)
    return e


def total_energy(config: Configuration, spec: LatticeSpec,
                 tables: KernelTables | None = None) -> int:
    """Exact exchange energy of one configuration.

    Uniform periodic lattices: E = -J (2 En - B) with En the aligned bonds,
    counted by the word kernels exactly as lattice.py:236-261 does.  Other
    lattices: E = |J| (2 e_idx - B) with e_idx the unsatisfied bonds.
    """
    if not spec.uniform:
        e_idx = unsatisfied_bonds(spec, config.index)
        unit = 2 * e_idx - spec.num_bonds
        scale = abs(spec.coupling)
        return unit if scale == 1 else scale * unit
    words, pairs = config.words, spec.word_neighbor_pairs()
    if tables is None:
        # direct bit counting (columns taller than the table cap)
        h = spec.rows
        misaligned = sum(popcount(w ^ circular_shift(w, h)) for w in words)
        misaligned += sum(popcount(words[a] ^ words[b]) for a, b in pairs)
        aligned = h * (len(words) + len(pairs)) - misaligned
    else:
        aligned = (sum(aligned_column_bonds(w, tables) for w in words) +
                   sum(aligned_row_bonds(words[a], words[b], tables)
                       for a, b in pairs))
    return -spec.coupling * (2 * aligned - spec.num_bonds)


def random_bond_signs(spec: LatticeSpec, seed: int, p_plus: float = 0.5):
    """i.i.d. +/-1 bond signs: the convention frozen for BASELINE config 4.

    ``numpy.random.default_rng(seed).random(B) < p_plus`` gives +1, drawn in
    bond_list() order.  The c4 draw (6x6 periodic, seed
    1234) is also committed as a fixture (tests/golden/c4_bond_signs.json).
    """
    base = LatticeSpec(spec.rows, spec.cols, spec.depth, spec.coupling,
                       boundary=spec.boundary)
    draws = np.random.default_rng(seed).random(base.num_bonds)
    return tuple(1 if x < p_plus else -1 for x in draws)
