"""Multi-GPU enumeration: one process per GPU, index-space shards, one reduce.

The reference parallelises with a `multiprocessing.Pool` of shard workers
and a root-side sum of the int64 tables (enumeration.py:356-390); the paper
does the same with MPI.  Here each rank of a
`torch.distributed` job (launched with torchrun, one process per GPU,
backend "nccl") walks `make_shards(spec, world)[rank]` — for a power-of-two
world exactly the top log2(P) bits of the index — into a device-resident
uint64 table, and a single `reduce` (sum) over NVLink combines the tables
on the root.  (Inside one process, `full_dos_timed` drives several GPUs
through the engine's own multi-device entry instead, which combines the
tables on the root with one peer-gather kernel.)  The table is at most 41 x 121 x 8 B = 39 KB, so the exchange
is one latency-bound message per walk (tens of microseconds against
milliseconds of enumeration); a fused kernel-side exchange would not pay
for itself here.

The per-rank enumeration function is a parameter only so that the CPU
tests can drive this host logic with the gloo backend; the default is the
native K1 engine and there is no CPU path in the product.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .enumeration import DoSHistogram, Shard, make_shards, native_lattice
from .lattice import LatticeSpec


def rank_shard(spec: LatticeSpec, rank: int, world: int) -> Shard:
    """The contiguous index range of `rank` (enumeration.py:44-63 partition)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    return make_shards(spec, world)[rank]


def native_enumerate_into(spec: LatticeSpec, shard: Shard, table) -> int:
    """K1 over `shard` into the CUDA int64 tensor `table`, on the current
    stream of the table's own device (the library launches on the calling
    thread's current device, so that device is made current first)."""
    import torch
    with torch.cuda.device(table.device):
        stream = torch.cuda.current_stream(table.device).cuda_stream
        return _native.enumerate_device(native_lattice(spec),
                                        shard.start_index, shard.end_index,
                                        table.data_ptr(), stream,
                                        accumulate=False)


def sharded_table(spec: LatticeSpec, group=None, root: int = 0,
                  enumerate_into=None, device=None):
    """Enumerate this rank's shard and reduce all tables onto `root` (a rank
    of `group`).

    Returns the reduced table tensor on every rank (only the root's holds
    the full sum).  Collective: every rank of `group` must call it.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    n, b = spec.num_spins, spec.num_bonds
    table = torch.zeros((n + 1) * (b + 1), dtype=torch.int64, device=device)
    fn = enumerate_into or native_enumerate_into
    fn(spec, rank_shard(spec, rank, world), table)
    if world > 1:
        # `root` is a rank of `group`; reduce takes a global rank
        dst = dist.get_global_rank(group, root) if group is not None else root
        dist.reduce(table, dst=dst, group=group)
    return table


def sharded_full_dos(spec: LatticeSpec, group=None, root: int = 0,
                     enumerate_into=None, device=None):
    """`full_dos` across the ranks of a process group.

    The root returns the complete DoSHistogram; other ranks return None.
    """
    import torch.distributed as dist

    table = sharded_table(spec, group, root, enumerate_into, device)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if rank != root:
        return None
    counts = table.cpu().numpy().reshape(spec.num_spins + 1,
                                         spec.num_bonds + 1)
    return DoSHistogram(spec, np.ascontiguousarray(counts))
