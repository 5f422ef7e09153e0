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
        for name in ("rows", "cols", "depth"):
            v = getattr(self, name)
            if not isinstance(v, int) or isinstance(v, bool):
                raise ValueError(f"{name} must be an integer, got {v!r}")
        if self.rows < 2 or self.cols < 2:
            raise ValueError(
                f"degenerate periodic axis: rows and cols must be >= 2, "
                f"got rows={self.rows} cols={self.cols}"
            )
        if self.depth < 1:
            raise ValueError(f"depth must be >= 1, got {self.depth}")
        if self.rows > MAX_ROWS:
            raise ValueError(f"rows={self.rows} exceeds the cap of {MAX_ROWS}")
        n = self.rows * self.cols * self.depth
        if n > MAX_SPINS:
            raise ValueError(
                f"{n} spins exceeds the cap of {MAX_SPINS} "
                f"(2^N must fit a 64-bit index with headroom)"
            )
        if self.coupling == 0:
            raise ValueError("coupling J must be nonzero")
        j = self.coupling
        if isinstance(j, float) and j.is_integer():
            object.__setattr__(self, "coupling", int(j))
        if self.boundary not in BOUNDARIES:
            raise ValueError(
                f"boundary must be one of {BOUNDARIES}, got {self.boundary!r}")
        if self.bond_signs is not None:
            signs = tuple(self.bond_signs)
            if len(signs) != self.num_bonds:
                raise ValueError(
                    f"bond_signs has {len(signs)} entries, lattice has "
                    f"{self.num_bonds} bonds")
            for s in signs:
                if isinstance(s, bool) or s not in (1, -1):
                    raise ValueError(f"bond signs must be +1 or -1, got {s!r}")
            object.__setattr__(self, "bond_signs",
                               tuple(int(s) for s in signs))

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
        """Inter-word bond pairs along cols (and layers in 3D).

        Same order as lattice.py:102-119; free boundaries omit the wrap
        pairs.  A periodic axis of length 2 lists both orders (double bond).
        """
        pairs = []
        for layer in range(self.depth):
            base = layer * self.cols
            for c in range(self.cols):
                if self.periodic or c + 1 < self.cols:
                    pairs.append((base + c, base + (c + 1) % self.cols))
        if self.depth > 1:
            for layer in range(self.depth):
                for c in range(self.cols):
                    if self.periodic or layer + 1 < self.depth:
                        pairs.append((layer * self.cols + c,
                                      ((layer + 1) % self.depth) * self.cols
                                      + c))
        return pairs

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
    if not 0 <= index < spec.num_configs:
        raise ValueError(f"index {index} outside [0, 2^{spec.num_spins})")
    mask = spec.word_mask
    words = tuple((index >> (w * spec.rows)) & mask
                  for w in range(spec.num_words))
    return Configuration(index=index, words=words)


def encode_words(spec: LatticeSpec, words) -> int:
    """Inverse of decode_config (lattice.py:140-148)."""
    if len(words) != spec.num_words:
        raise ValueError(f"expected {spec.num_words} words, got {len(words)}")
    index = 0
    for w, word in enumerate(words):
        if not 0 <= word <= spec.word_mask:
            raise ValueError(
                f"word {word:#x} has stray bits above row {spec.rows}")
        index |= word << (w * spec.rows)
    return index


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
    words = config.words
    if tables is not None:
        aligned = sum(aligned_column_bonds(w, tables) for w in words)
        aligned += sum(aligned_row_bonds(words[a], words[b], tables)
                       for a, b in spec.word_neighbor_pairs())
    else:
        rows = spec.rows
        aligned = sum(rows - popcount(w ^ circular_shift(w, rows))
                      for w in words)
        aligned += sum(rows - popcount(words[a] ^ words[b])
                       for a, b in spec.word_neighbor_pairs())
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
