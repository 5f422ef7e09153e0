"""World-size-2 test of the sharded driver's host logic on CPU (gloo).

The multi-GPU path (paper_1110_2561_b200.distributed) shards the index
space by rank and reduces the per-rank tables onto the root.  Here the two
ranks are CPU processes with the gloo backend, and each rank's enumeration
is the oracle port (test injection) — so this covers the partition, the
collective and the root assembly, not the kernel (the GPU tests do that).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, tcp_port, kw, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1110_2561_b200 as isd
    from paper_1110_2561_b200 import distributed as D
    from oracle import port

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{tcp_port}",
                            rank=rank, world_size=world)
    spec = isd.LatticeSpec(**kw)

    def oracle_into(spec, shard, table):
        lat = port.Lattice(spec.rows, spec.cols, spec.depth, spec.coupling,
                           spec.periodic)
        t = port.enumerate_range(lat, shard.start_index, shard.end_index)
        table.copy_(torch.from_numpy(t.reshape(-1)))
        return 0

    dos = D.sharded_full_dos(spec, enumerate_into=oracle_into,
                             device=torch.device("cpu"))
    if rank == 0:
        np.save(out_path, dos.counts)
    else:
        assert dos is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kw,world", [(dict(rows=4, cols=4), 2),
                                      (dict(rows=3, cols=3, depth=2), 2),
                                      (dict(rows=3, cols=5), 3)])
def test_two_rank_gloo_reduce_equals_single_walk(tmp_path, kw, world):
    from oracle import port
    out = str(tmp_path / "table.npy")
    mp.start_processes(_worker, args=(world, _free_port(), kw, out),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    lat = port.Lattice(kw["rows"], kw["cols"], kw.get("depth", 1))
    want = port.enumerate_range(lat, 0, 1 << lat.n)
    assert np.array_equal(got, want)


def test_rank_shards_are_top_bits_for_power_of_two():
    import paper_1110_2561_b200 as isd
    from paper_1110_2561_b200.distributed import rank_shard
    spec = isd.LatticeSpec(3, 3, 4)
    for world in (2, 4, 8):
        bits = world.bit_length() - 1
        for r in range(world):
            sh = rank_shard(spec, r, world)
            assert sh.start_index == r << (36 - bits)
            assert sh.size == 1 << (36 - bits)
    with pytest.raises(ValueError):
        rank_shard(spec, 2, 2)


def _subgroup_worker(rank, world, tcp_port, kw, out_path):
    # ranks 1 and 2 form a subgroup whose root is its group rank 1 (global
    # rank 2): the reduce must target the global rank of the group's root
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1110_2561_b200 as isd
    from paper_1110_2561_b200 import distributed as D
    from oracle import port

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{tcp_port}",
                            rank=rank, world_size=world)
    sub = dist.new_group([1, 2])
    spec = isd.LatticeSpec(**kw)

    def oracle_into(spec, shard, table):
        lat = port.Lattice(spec.rows, spec.cols, spec.depth, spec.coupling,
                           spec.periodic)
        t = port.enumerate_range(lat, shard.start_index, shard.end_index)
        table.copy_(torch.from_numpy(t.reshape(-1)))
        return 0

    if rank in (1, 2):
        dos = D.sharded_full_dos(spec, group=sub, root=1,
                                 enumerate_into=oracle_into,
                                 device=torch.device("cpu"))
        if rank == 2:
            np.save(out_path, dos.counts)
        else:
            assert dos is None
    dist.barrier()
    dist.destroy_process_group()


def test_subgroup_root_is_a_group_rank(tmp_path):
    from oracle import port
    out = str(tmp_path / "table.npy")
    kw = dict(rows=3, cols=4)
    mp.start_processes(_subgroup_worker, args=(3, _free_port(), kw, out),
                       nprocs=3, join=True, start_method="spawn")
    lat = port.Lattice(3, 4, 1)
    assert np.array_equal(np.load(out), port.enumerate_range(lat, 0, 1 << 12))
