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

from .enumeration import full_dos_timed
from .lattice import LatticeSpec

REPORT_HEADER = "rows,cols,depth,N,workers,wall_seconds,speedup"
# report column -> parser, in column order
_REPORT_COLUMNS = (("rows", int), ("cols", int), ("depth", int), ("N", int),
                   ("workers", int), ("wall_seconds", float),
                   ("speedup", float))


class ResultMismatchError(RuntimeError):
    """A benchmarked run produced a histogram different from the baseline."""


@dataclass
class BenchRecord:
    spec: LatticeSpec
    num_workers: int
    wall_seconds: float
    per_worker_seconds: list[float] = field(default_factory=list)
    speedup_vs_one: float = 0.0
    configs_per_second: float = 0.0


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


def run_bench(spec: LatticeSpec, worker_counts, repeats: int = 3):
    counts = list(worker_counts)
    _check_arguments(counts, repeats)
    expected, single_wall, _ = full_dos_timed(spec, workers=1)
    records = []
    for shards in counts:
        wall, per_shard = _fastest_walk(spec, shards, repeats, expected)
        records.append(BenchRecord(spec, shards, wall, per_shard,
                                   configs_per_second=spec.num_configs / wall))
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


def parse_scaling_report(text: str) -> list[dict]:
    rows = [ln for ln in text.splitlines() if ln.strip()]
    if not rows or rows[0] != REPORT_HEADER:
        raise ValueError(f"expected header {REPORT_HEADER!r}")
    parsed = []
    for row in rows[1:]:
        cells = row.split(",")
        if len(cells) != len(_REPORT_COLUMNS):
            raise ValueError(f"malformed report row {row!r}")
        parsed.append({name: cast(cell) for (name, cast), cell
                       in zip(_REPORT_COLUMNS, cells)})
    return parsed
