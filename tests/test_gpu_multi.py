"""GPU tests of the engine-side multi-device walk and of the robustness fixes.

`isd_enumerate_multi` splits a walk into shards with the reference's
partition (make_shards, enumeration.py:44-63), walks shard i on devs[i] and
combines the per-device tables on the root with one peer-gather kernel
(enumeration.py:365-390's Pool + root sum, on the device).  On the one-GPU
pool every shard is listed on device 0, which runs them one after another
and times each alone — the same code path as P GPUs minus the NVLink reads.
Integer tables must be bit-exact against the reference's goldens.
"""

import numpy as np
import pytest

import paper_1110_2561_b200 as isd
from paper_1110_2561_b200 import _native
from paper_1110_2561_b200.enumeration import native_lattice
from paper_1110_2561_b200.workloads import workloads
from golden_io import read_csv_table

pytestmark = pytest.mark.gpu


def golden(name):
    rows, cols, depth, j, table = read_csv_table(name)
    return isd.LatticeSpec(rows, cols, depth, j), table


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_multi_walk_of_c5_equals_reference_golden(shards):
    spec, want = golden("dos_3x3x4_J1.csv")
    table, shard_ms, total_ms = _native.enumerate_multi(
        native_lattice(spec), 0, spec.num_configs, [0] * shards)
    assert np.array_equal(table.view(np.int64), want)
    assert len(shard_ms) == shards and all(ms > 0 for ms in shard_ms)
    # the root's span covers every shard (all ran on this one device)
    assert total_ms >= sum(shard_ms) * 0.99


def test_multi_walk_device_copy_path():
    # where the root has no peer access it copies each device's table
    # (cudaMemcpyPeerAsync) before the gather: forced here on one device
    spec, want = golden("dos_5x5x1_J1.csv")
    with _native.knobs(ISD_PEER=0):
        table, _, _ = _native.enumerate_multi(
            native_lattice(spec), 0, spec.num_configs, [0, 0, 0])
    assert np.array_equal(table.view(np.int64), want)


@pytest.mark.parametrize("shards", [1, 4, 5])
def test_multi_walk_with_flip_symmetry(shards):
    spec, want = golden("dos_3x3x4_J1.csv")
    algo = _native.ALGO_AUTO | _native.FLAG_FLIP_SYMMETRY
    table, shard_ms, _ = _native.enumerate_multi(
        native_lattice(spec), 0, spec.num_configs, [0] * shards, algo)
    assert np.array_equal(table.view(np.int64), want)


@pytest.mark.parametrize("name,shards", [
    ("dos_4x4x1_J1.csv", 7), ("dos_5x5x1_J1.csv", 3),
    ("dos_5x5x1_J1.csv", 64), ("dos_2x2x1_J1.csv", 16),
    ("dos_6x6x1_J1.csv", 8)])
def test_multi_walk_small_lattices_any_shard_count(name, shards):
    spec, want = golden(name)
    table, shard_ms, _ = _native.enumerate_multi(
        native_lattice(spec), 0, spec.num_configs, [0] * shards)
    assert np.array_equal(table.view(np.int64), want)
    assert len(shard_ms) == shards


def test_multi_walk_of_a_sub_range_equals_single_walk():
    spec = isd.LatticeSpec(5, 5)
    lat = native_lattice(spec)
    a, b = 123457, 123457 + (1 << 22) + 999
    one, _ = _native.enumerate_host(lat, a, b)
    many, _, _ = _native.enumerate_multi(lat, a, b, [0] * 5)
    assert np.array_equal(one, many)


def test_multi_walk_validates_arguments():
    spec = isd.LatticeSpec(2, 2)  # 16 configurations
    lat = native_lattice(spec)
    with pytest.raises(ValueError, match="shards"):
        _native.enumerate_multi(lat, 0, 16, [0] * 17)
    with pytest.raises(ValueError, match="invalid"):
        _native.enumerate_multi(lat, 0, 17, [0])
    with pytest.raises(_native.NativeError, match="device"):
        _native.enumerate_multi(lat, 0, 16, [0, 99])
    with pytest.raises(ValueError, match="full range"):
        _native.enumerate_multi(lat, 0, 8, [0],
                                _native.FLAG_FLIP_SYMMETRY)


def test_full_dos_timed_uses_the_multi_walk():
    spec, want = golden("dos_3x3x4_J1.csv")
    dos, wall, per = isd.full_dos_timed(spec, workers=4)
    assert np.array_equal(dos.counts, want)
    assert len(per) == 4 and all(p > 0 for p in per) and wall > 0
    # each shard is a quarter of the walk: its own device time, not the sum
    assert max(per) < wall


def test_thermo_gather_fuses_the_table_sum():
    torch = pytest.importorskip("torch")
    w = workloads()["c2"]
    spec = w.spec
    lat = native_lattice(spec)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev).cuda_stream
    nb = (spec.num_spins + 1) * (spec.num_bonds + 1)
    shards = isd.make_shards(spec, 5)
    parts = [torch.zeros(nb, dtype=torch.int64, device=dev) for _ in shards]
    for sh, t in zip(shards, parts):
        _native.enumerate_device(lat, sh.start_index, sh.end_index,
                                 t.data_ptr(), st)
    fields = torch.tensor(w.fields, dtype=torch.float64, device=dev)
    temps = torch.tensor(w.temps, dtype=torch.float64, device=dev)
    npts = len(w.fields) * len(w.temps)
    out = torch.empty(npts * 7, dtype=torch.float64, device=dev)
    total = torch.empty(nb, dtype=torch.int64, device=dev)
    _native.thermo_gather_device([t.data_ptr() for t in parts],
                                 total.data_ptr(), spec.num_spins,
                                 spec.num_bonds, abs(spec.coupling),
                                 fields.data_ptr(), len(w.fields),
                                 temps.data_ptr(), len(w.temps),
                                 out.data_ptr(), st)
    torch.cuda.synchronize(dev)
    whole = isd.full_dos(spec)
    assert np.array_equal(total.cpu().numpy().reshape(whole.counts.shape),
                          whole.counts)
    ref = isd.thermo_grid(whole, w.fields, w.temps)
    got = out.cpu().numpy().reshape(len(w.fields), len(w.temps), 7)
    # same kernel over the same table: identical, not merely close
    assert np.array_equal(got, ref)
    # gather only (no grid): one kernel forms the sum
    total.zero_()
    _native.thermo_gather_device([t.data_ptr() for t in parts],
                                 total.data_ptr(), spec.num_spins,
                                 spec.num_bonds, 1.0, 0, 0, 0, 0, 0, st)
    torch.cuda.synchronize(dev)
    assert np.array_equal(total.cpu().numpy().reshape(whole.counts.shape),
                          whole.counts)


def test_small_grid_cannot_wrap_shared_counters():
    # a 2-SM grid walks 2^36 configurations: the launch cap derived from the
    # grid (2^31 per SM) keeps every CTA's u32 counters below 2^32
    spec, want = golden("dos_3x3x4_J1.csv")
    with _native.knobs(ISD_GRID_SMS=2, ISD_AUTOTUNE=0):
        table, _ = _native.enumerate_host(native_lattice(spec), 0,
                                          spec.num_configs)
    assert np.array_equal(table.view(np.int64), want)


def test_first_large_walk_inside_graph_capture():
    # the first walk of a plan key is normally autotuned (synchronous timing
    # launches): inside a stream capture the model's plan is used instead
    torch = pytest.importorskip("torch")
    spec = workloads()["c3"].spec
    lat = native_lattice(spec)
    dev = torch.device("cuda", 0)
    nb = (spec.num_spins + 1) * (spec.num_bonds + 1)
    table = torch.zeros(nb, dtype=torch.int64, device=dev)
    cap = torch.cuda.Stream(dev)
    g = torch.cuda.CUDAGraph()
    # a knob set no other test uses: a plan key with no tuned entry
    with _native.knobs(ISD_TUNE_CANDIDATES=39):
        with torch.cuda.graph(g, stream=cap):
            _native.enumerate_device(lat, 0, 1 << 33, table.data_ptr(),
                                     cap.cuda_stream)
        g.replay()
        torch.cuda.synchronize(dev)
    want, _ = _native.enumerate_host(lat, 0, 1 << 33)
    assert np.array_equal(table.cpu().numpy().reshape(want.shape),
                          want.view(np.int64))


def test_calls_restore_the_callers_current_device():
    torch = pytest.importorskip("torch")
    torch.cuda.set_device(0)
    spec = isd.LatticeSpec(4, 4)
    isd.enumerate_shard(spec, None, isd.make_shards(spec, 1)[0], device=0)
    assert torch.cuda.current_device() == 0


def test_knobs_are_not_read_from_the_environment(monkeypatch):
    # ISD_JIT=2 would force the NVRTC kernel on a small walk if the library
    # read the environment; it does not
    monkeypatch.setenv("ISD_JIT", "2")
    spec = isd.LatticeSpec(5, 5)
    isd.full_dos(spec)
    assert _native.kernel_info() == "k1_hoisted_aot"
    with _native.knobs(ISD_JIT=2):
        isd.full_dos(spec)
        assert _native.kernel_info() == "k1_hoisted_jit"


@pytest.mark.parametrize("name,workers,flip", [("c2", 1, False), ("c2", 5, False),
                                               ("c5", 8, False), ("c5", 4, True),
                                               ("c1", 3, False)])
def test_dos_thermo_equals_full_dos_then_thermo_grid(name, workers, flip):
    w = workloads()[name]
    dos, grid = isd.dos_thermo(w.spec, w.fields, w.temps, workers,
                               flip_symmetry=flip)
    want = isd.full_dos(w.spec)
    assert dos == want
    # the same K2 over the same table: identical, not merely close
    assert np.array_equal(grid, isd.thermo_grid(want, w.fields, w.temps))


def test_dos_thermo_validates():
    spec = isd.LatticeSpec(3, 3)
    with pytest.raises(ValueError, match="temperature"):
        isd.dos_thermo(spec, [0.0], [1.0, 0.0])
    with pytest.raises(ValueError, match="workers"):
        isd.dos_thermo(spec, [0.0], [1.0], workers=0)
    dos, grid = isd.dos_thermo(spec, [], [1.0])
    assert grid.shape == (0, 1, 7) and dos == isd.full_dos(spec)
