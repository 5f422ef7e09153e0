"""Scaling harness over shard counts.

Mirrors /root/reference/pkg/src/isingdos/bench.py: min-of-repeats wall
time per shard count, a hard identity check of every run against the
1-shard result (`ResultMismatchError`), and the same CSV report
(`rows,cols,depth,N,workers,wall_seconds,speedup`).  Here a "worker" is a
shard mapped onto the visible GPUs by `full_dos_timed`; records add the
configurations/s and the per-shard device time.  `full_dos_timed` is looked
up as a module global, as in the reference (bench.py:10, 52, 59), so tests
can substitute it.
"""

from dataclasses import dataclass, field

from .enumeration import full_dos_timed
from .lattice import LatticeSpec


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


def run_bench(spec: LatticeSpec, worker_counts, repeats: int = 3):
    counts = list(worker_counts)
    if not counts:
        raise ValueError("worker_counts must be nonempty")
    if any(not isinstance(p, int) or p < 1 for p in counts):
        raise ValueError(f"worker counts must be positive integers: {counts}")
    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")
    reference, ref_wall, _ = full_dos_timed(spec, workers=1)
    records = []
    for p in counts:
        best_wall = best_per = None
        for _ in range(repeats):
            hist, wall, per_worker = full_dos_timed(spec, workers=p)
            if hist != reference:
                raise ResultMismatchError(
                    f"{p}-worker run disagrees with the 1-worker result "
                    f"on {spec.rows}x{spec.cols}x{spec.depth}")
            if best_wall is None or wall < best_wall:
                best_wall, best_per = wall, per_worker
        records.append(BenchRecord(
            spec=spec, num_workers=p, wall_seconds=best_wall,
            per_worker_seconds=best_per,
            configs_per_second=spec.num_configs / best_wall))
    baseline = next((r.wall_seconds for r in records if r.num_workers == 1),
                    ref_wall)
    for r in records:
        r.speedup_vs_one = baseline / r.wall_seconds
    return records


REPORT_HEADER = "rows,cols,depth,N,workers,wall_seconds,speedup"


def emit_scaling_report(records) -> str:
    records = list(records)
    if not records:
        raise ValueError("no records to report")
    rows = [REPORT_HEADER]
    for r in sorted(records, key=lambda r: (r.spec.num_spins, r.num_workers)):
        s = r.spec
        rows.append(f"{s.rows},{s.cols},{s.depth},{s.num_spins},"
                    f"{r.num_workers},{r.wall_seconds!r},{r.speedup_vs_one!r}")
    return "\n".join(rows) + "\n"


def parse_scaling_report(text: str) -> list[dict]:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != REPORT_HEADER:
        raise ValueError(f"expected header {REPORT_HEADER!r}")
    out = []
    for ln in lines[1:]:
        rows, cols, depth, n, workers, wall, speedup = ln.split(",")
        out.append({"rows": int(rows), "cols": int(cols), "depth": int(depth),
                    "N": int(n), "workers": int(workers),
                    "wall_seconds": float(wall), "speedup": float(speedup)})
    return out
