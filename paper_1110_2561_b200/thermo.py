"""Exact thermodynamics from g(M, E) at any field and temperature, on B200.

Drop-in for /root/reference/pkg/src/isingdos/thermo.py.  `partition_point`
and `thermo_sweep` keep their signatures, validation and error messages
(thermo.py:46-63, 91-100); the arithmetic (max-shifted log-sum-exp over
occupied cells, central second moments, thermo.py:65-77) runs in the fp64
K2 kernel, one CTA per (h, T) point, so a sweep is one launch and every
point is computed by the same code whatever grid it belongs to.
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from .enumeration import DoSHistogram


@dataclass(frozen=True)
class ThermoPoint:
    """Observables of one (h, T) evaluation (thermo.py:16-34).

    mean_abs_magnetization <|M|> is an extension (BASELINE configs 2, 5);
    it comes last and has a default so the reference's 8 positional fields
    are unchanged.
    """

    field: float
    temperature: float
    log_z: float
    free_energy: float
    internal_energy: float
    specific_heat: float
    mean_magnetization: float
    susceptibility: float
    mean_abs_magnetization: float = float("nan")


def _check_complete(dos: DoSHistogram) -> None:
    if dos.total() != dos.spec.num_configs:
        raise ValueError(
            f"histogram total {dos.total()} != 2^{dos.spec.num_spins}; "
            f"not a complete density of states")


def thermo_grid(dos: DoSHistogram, fields, temps, *, device=None):
    """All observables on a (field x temperature) grid in one launch.

    Returns float64 array [len(fields), len(temps), 7] with columns
    log_z, free_energy, internal_energy, specific_heat, mean_magnetization,
    susceptibility, mean_abs_magnetization.
    """
    fields = np.asarray(fields, dtype=np.float64).reshape(-1)
    temps = np.asarray(temps, dtype=np.float64).reshape(-1)
    if not np.all(temps > 0):  # (NaN fails too)
        raise ValueError("all temperatures must be > 0")
    _check_complete(dos)
    spec = dos.spec
    counts = np.ascontiguousarray(dos.counts).view(np.uint64)
    out, _ = _native.thermo_host(counts, spec.num_spins, spec.num_bonds,
                                 float(dos.energy_scale), fields, temps,
                                 device=device)
    return out


def dos_thermo(spec, fields, temps, workers=None, *, flip_symmetry=False):
    """Density of states and its thermodynamic grid in one engine call
    (an extension: `full_dos` + `thermo_grid` without the table's round
    trip through the host).

    The shards (as `full_dos_timed`: `workers`, default one per GPU) are
    walked and combined on the root GPU, which then evaluates the
    (fields x temps) grid from the combined table; one synchronisation.
    Returns (DoSHistogram, float64 array [len(fields), len(temps), 7]) with
    the columns of `thermo_grid`.
    """
    from .enumeration import (_plan_shards, _signed, gpu_count,
                              native_lattice)
    fields = np.asarray(fields, dtype=np.float64).reshape(-1)
    temps = np.asarray(temps, dtype=np.float64).reshape(-1)
    if not np.all(temps > 0):  # (NaN fails too)
        raise ValueError("all temperatures must be > 0")
    if workers is None:
        workers = min(max(gpu_count(), 1), spec.num_configs)
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    shards = _plan_shards(spec, workers, flip_symmetry)
    devices = gpu_count()
    if devices < 1:
        raise _native.NativeError("no CUDA device available for enumeration")
    algo = _native.ALGO_AUTO | (_native.FLAG_FLIP_SYMMETRY if flip_symmetry
                                else 0)
    table, grid, _, _ = _native.enumerate_thermo(
        native_lattice(spec), 0, spec.num_configs,
        [sh.shard_id % devices for sh in shards], abs(spec.coupling),
        fields, temps, algo)
    return DoSHistogram(spec, _signed(table)), grid


def _point(h, t, row) -> ThermoPoint:
    return ThermoPoint(field=h, temperature=t, log_z=float(row[0]),
                       free_energy=float(row[1]),
                       internal_energy=float(row[2]),
                       specific_heat=float(row[3]),
                       mean_magnetization=float(row[4]),
                       susceptibility=float(row[5]),
                       mean_abs_magnetization=float(row[6]))


def partition_point(dos: DoSHistogram, h: float,
                    temperature: float) -> ThermoPoint:
    """log Z and the standard observables at one (h, T) (thermo.py:46-88).

    Raises:
        ValueError: for T <= 0 or an incomplete histogram.
    """
    if temperature <= 0:
        raise ValueError(f"temperature must be > 0, got {temperature}")
    _check_complete(dos)
    out = thermo_grid(dos, [h], [temperature])
    return _point(h, temperature, out[0, 0])


def thermo_sweep(dos: DoSHistogram, h: float, temps) -> list[ThermoPoint]:
    """partition_point at each temperature of a strictly increasing grid."""
    temps = list(temps)
    if not temps:
        raise ValueError("temperature list must be nonempty")
    if any(t <= 0 for t in temps):
        raise ValueError("all temperatures must be > 0")
    if any(b <= a for a, b in zip(temps, temps[1:])):
        raise ValueError("temperatures must be strictly increasing")
    _check_complete(dos)
    out = thermo_grid(dos, [h], temps)
    return [_point(h, t, out[0, i]) for i, t in enumerate(temps)]


def temperature_grid(tmin: float, tmax: float, tstep: float) -> list[float]:
    """T_i = tmin + i*tstep with the reference CLI's step count (cli.py:83-84)."""
    if tstep <= 0:
        raise ValueError(f"tstep must be > 0, got {tstep}")
    if tmax < tmin:
        raise ValueError(f"tmax {tmax} < tmin {tmin}")
    n_steps = int((tmax - tmin) / tstep + 1e-9) + 1
    return [tmin + i * tstep for i in range(n_steps)]
