"""The five BASELINE.json lattices and their thermodynamic grids.

c1..c5 follow BASELINE.json `configs` (and SURVEY.md §8d).  c4's bond
signs use the convention frozen in `lattice.random_bond_signs` (seed 1234,
numpy default_rng, bond_list order); tests/golden/c4_bond_signs.json holds
the same 72 signs as a fixture.
"""

from dataclasses import dataclass

from .lattice import LatticeSpec, random_bond_signs
from .thermo import temperature_grid


@dataclass(frozen=True)
class Workload:
    name: str
    spec: LatticeSpec
    fields: tuple
    tmin: float
    tmax: float
    tstep: float
    description: str

    @property
    def temps(self):
        return temperature_grid(self.tmin, self.tmax, self.tstep)


def _c4_spec():
    base = LatticeSpec(6, 6)
    return LatticeSpec(6, 6, bond_signs=random_bond_signs(base, 1234))


def workloads() -> dict:
    return {
        "c1": Workload("c1", LatticeSpec(4, 4, boundary="free"),
                       (0.0, 0.1, 0.5), 0.5, 5.0, 0.05,
                       "2D 4x4 free, N=16, J=+1"),
        "c2": Workload("c2", LatticeSpec(5, 5), (0.0,), 0.5, 5.0, 0.01,
                       "2D 5x5 periodic, N=25, J=+1"),
        "c3": Workload("c3", LatticeSpec(6, 6, boundary="free"),
                       (0.0, 0.05, 0.1), 0.5, 5.0, 0.01,
                       "2D 6x6 free, N=36, J=+1"),
        "c4": Workload("c4", _c4_spec(), (0.0,), 0.2, 4.0, 0.01,
                       "2D 6x6 periodic, N=36, +/-J seed 1234"),
        "c5": Workload("c5", LatticeSpec(3, 3, 4), (0.0, 0.1), 1.0, 8.0, 0.02,
                       "3D 3x3x4 periodic, N=36, J=+1"),
    }


# Canonical per-configuration integer work: W 32-bit words,
# C bond classes, L LOP3 per class (1 uniform, 2 with +/-J).
def canonical_ops(spec: LatticeSpec) -> tuple[int, int]:
    """(POPC ops, ALU ops) per configuration of the canonical formulation."""
    w = (spec.num_spins + 31) // 32
    c = len(spec.bond_classes())
    l = 1 if spec.bond_signs is None else 2
    return w * (1 + c), w * c * (2 + l) + (w - 1)
