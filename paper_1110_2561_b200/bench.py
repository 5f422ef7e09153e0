"""Scaling harness over shard counts.

Same contract as the reference harness (/root/reference/pkg/src/isingdos/
bench.py:29-95): for each shard count the fastest of `repeats` complete
walks is kept, every walk must reproduce the single-shard table exactly or
`ResultMismatchError` is raised, and the report is the CSV
``rows,cols,depth,N,workers,wall_seconds,speedup`` sorted by (N, workers)
with floats written losslessly.  On this engine a "worker" is one shard of
`full_dos_timed` spread over the visible GPUs, and each record also carries
the configurations/s of its best walk.  `full_dos_timed` is resolved as a
module global at call time (as the reference does) so tests can patch it.
"""

from dataclasses import dataclass, field

from . import _native
from .enumeration import full_dos_timed, gpu_count, native_lattice
from .lattice import LatticeSpec

REPORT_HEADER = "rows,cols,depth,N,workers,wall_seconds,speedup"
# report column -> parser, in column order
_REPORT_COLUMNS = (("rows", int), ("cols", int), ("depth", int), ("N", int),
                   ("workers", int), ("wall_seconds", float),
                   ("speedup", float))
# the extended report: the reference's columns, then the engine's own
EXTENDED_HEADER = (REPORT_HEADER +
                   ",gpus,configs_per_second,roofline_fraction,sm_mhz")
_EXTENDED_COLUMNS = _REPORT_COLUMNS + (
    ("gpus", int), ("configs_per_second", float),
    ("roofline_fraction", lambda x: None if x == "" else float(x)),
    ("sm_mhz", lambda x: None if x == "" else float(x)))


class ResultMismatchError(RuntimeError):
    """A benchmarked run produced a histogram different from the baseline."""


@dataclass
class BenchRecord:
    """One (lattice, shard count) measurement (reference bench.py:19-26),
    plus what the GPU run adds: the GPUs the shards ran on, the walk's
    configurations/s, the enumeration kernel's fraction of its measured
    roofline and the SM clock that roofline was measured at."""

    spec: LatticeSpec
    num_workers: int
    wall_seconds: float
    per_worker_seconds: list[float] = field(default_factory=list)
    speedup_vs_one: float = 0.0
    configs_per_second: float = 0.0
    num_gpus: int = 0
    roofline_fraction: float | None = None
    sm_clock_mhz: float | None = None


def _check_arguments(counts: list, repeats: int) -> None:
    if not counts:
        raise ValueError("worker_counts must be nonempty")
    bad = [p for p in counts if not isinstance(p, int) or p < 1]
    if bad:
        raise ValueError(f"worker counts must be positive integers: {counts}")
    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")


def _fastest_walk(spec: LatticeSpec, shards: int, repeats: int, expected):
    """Best (wall, per-shard times) of `repeats` verified walks."""
    trials = []
    for _ in range(repeats):
        table, wall, per_shard = full_dos_timed(spec, workers=shards)
        if table != expected:
            raise ResultMismatchError(
                f"{shards}-worker run disagrees with the 1-worker result "
                f"on {spec.rows}x{spec.cols}x{spec.depth}")
        trials.append((wall, per_shard))
    return min(trials, key=lambda t: t[0])


_PEAKS: dict = {}


def _red_peak(device: int):
    """(conflict-free shared RED lanes per second, SM MHz) of one GPU, from
    the engine's K0 probe (measured once per process)."""
    if device not in _PEAKS:
        lanes, mhz = _native.calibrate(3, device=device)
        _PEAKS[device] = (lanes * _native.sm_count(device) * mhz * 1e6, mhz)
    return _PEAKS[device]


def _roofline(spec: LatticeSpec, shards: int, per_shard: list[float]):
    """(GPUs used, mean fraction of the RED roofline over those GPUs, mean
    SM MHz) of one walk.  Shard i ran on GPU i mod #GPUs; a GPU's rate is
    its shards' configurations over their summed device time, its peak the
    K0 RED rate times the configurations one RED lane counts in the plan
    (2^pair_mode).  (None, None) without a probe."""
    gpus = max(1, min(shards, gpu_count()))
    try:
        size = spec.num_configs // shards
        _, plan = _native.plan(native_lattice(spec), max(size, 1))
        per_red = 1 << plan.pair_mode
        fracs, clocks = [], []
        edges = [i * spec.num_configs // shards for i in range(shards + 1)]
        for d in range(gpus):
            mine = [i for i in range(shards) if i % gpus == d]
            busy = sum(per_shard[i] for i in mine)
            work = sum(edges[i + 1] - edges[i] for i in mine)
            peak, mhz = _red_peak(d)
            fracs.append(work / busy / (peak * per_red))
            clocks.append(mhz)
        return gpus, sum(fracs) / len(fracs), sum(clocks) / len(clocks)
    except (_native.NativeError, ImportError, OSError, ZeroDivisionError):
        return gpus, None, None


def run_bench(spec: LatticeSpec, worker_counts, repeats: int = 3,
              roofline: bool = False):
    """The reference's scaling sweep (bench.py:29-95).  With `roofline`,
    each record also gets the kernel's roofline fraction and the SM clock
    (one K0 probe per GPU)."""
    counts = list(worker_counts)
    _check_arguments(counts, repeats)
    expected, single_wall, _ = full_dos_timed(spec, workers=1)
    records = []
    for shards in counts:
        wall, per_shard = _fastest_walk(spec, shards, repeats, expected)
        rec = BenchRecord(spec, shards, wall, per_shard,
                          configs_per_second=spec.num_configs / wall)
        if roofline:
            rec.num_gpus, rec.roofline_fraction, rec.sm_clock_mhz = \
                _roofline(spec, shards, per_shard)
        else:
            rec.num_gpus = max(1, min(shards, gpu_count()))
        records.append(rec)
    # speed-ups are relative to the measured 1-shard point when the sweep
    # has one, else to the verification walk
    ones = [r.wall_seconds for r in records if r.num_workers == 1]
    base = ones[0] if ones else single_wall
    for r in records:
        r.speedup_vs_one = base / r.wall_seconds
    return records


def emit_scaling_report(records) -> str:
    ordered = sorted(records, key=lambda r: (r.spec.num_spins, r.num_workers))
    if not ordered:
        raise ValueError("no records to report")
    body = []
    for r in ordered:
        fields = (r.spec.rows, r.spec.cols, r.spec.depth, r.spec.num_spins,
                  r.num_workers, repr(r.wall_seconds), repr(r.speedup_vs_one))
        body.append(",".join(str(f) for f in fields))
    return "\n".join([REPORT_HEADER] + body) + "\n"


def emit_extended_report(records) -> str:
    """The reference CSV with four more columns per record: gpus,
    configs_per_second, roofline_fraction, sm_mhz (empty when unmeasured)."""
    ordered = sorted(records, key=lambda r: (r.spec.num_spins, r.num_workers))
    if not ordered:
        raise ValueError("no records to report")

    def opt(x):
        return "" if x is None else repr(float(x))

    body = []
    for r in ordered:
        fields = (r.spec.rows, r.spec.cols, r.spec.depth, r.spec.num_spins,
                  r.num_workers, repr(r.wall_seconds), repr(r.speedup_vs_one),
                  r.num_gpus, repr(float(r.configs_per_second)),
                  opt(r.roofline_fraction), opt(r.sm_clock_mhz))
        body.append(",".join(str(f) for f in fields))
    return "\n".join([EXTENDED_HEADER] + body) + "\n"


def parse_scaling_report(text: str) -> list[dict]:
    """Parse either report (the header says which)."""
    rows = [ln for ln in text.splitlines() if ln.strip()]
    if not rows or rows[0] not in (REPORT_HEADER, EXTENDED_HEADER):
        raise ValueError(f"expected header {REPORT_HEADER!r}")
    columns = _REPORT_COLUMNS if rows[0] == REPORT_HEADER else \
        _EXTENDED_COLUMNS
    parsed = []
    for row in rows[1:]:
        cells = row.split(",")
        if len(cells) != len(columns):
            raise ValueError(f"malformed report row {row!r}")
        parsed.append({name: cast(cell) for (name, cast), cell
                       in zip(columns, cells)})
    return parsed
