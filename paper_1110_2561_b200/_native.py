"""ctypes binding of the C ABI in include/isingdos_b200.h.

This is the only place Python touches the native engine.  There is no CPU
fallback: if the library is missing the import of any compute entry point
raises, and if no GPU is present the compute calls raise RuntimeError with
the library's own message.
"""

import contextlib
import ctypes
import os
import threading

import numpy as np

from ._build import LIB

ISD_MAX_CLASSES = 8
ISD_COPY_BITS = 7
ISD_THERMO_FIELDS = 7

ALGO_AUTO = 0
ALGO_CANONICAL = 1
ALGO_HOISTED = 2
FLAG_FLIP_SYMMETRY = 0x100

EXPORTED_SYMBOLS = (
    "isd_enumerate", "isd_enumerate_async", "isd_thermo", "isd_thermo_async",
    "isd_plan", "isd_validate", "isd_calibrate", "isd_device_count",
    "isd_sm_count", "isd_last_error", "isd_version", "isd_abi_version",
    "isd_launch_count", "isd_mirror_async", "isd_kernel_info",
    "isd_jit_check", "isd_band_items", "isd_set_knob", "isd_clear_knobs",
    "isd_set_cache_dirs", "isd_build_id", "isd_enumerate_multi",
    "isd_thermo_gather_async", "isd_walk_plan", "isd_set_walk_plan",
    "isd_band_costs", "isd_plan_range", "isd_naive_enumerate",
    "isd_enumerate_thermo", "isd_band_slot_order",
)


class BondClass(ctypes.Structure):
    _fields_ = [("shift", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("bond_mask", ctypes.c_uint64), ("jneg_mask", ctypes.c_uint64)]


class Lattice(ctypes.Structure):
    _fields_ = [("n_spins", ctypes.c_uint32), ("n_bonds", ctypes.c_uint32),
                ("n_classes", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("classes", BondClass * ISD_MAX_CLASSES)]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("u", ctypes.c_uint32), ("l", ctypes.c_uint32), ("k", ctypes.c_uint32),
        ("stride", ctypes.c_uint32),
        ("run_mask_above_k", ctypes.c_uint64), ("loop_mask", ctypes.c_uint64),
        ("copy_site", ctypes.c_int32 * ISD_COPY_BITS),
        ("copy_degree", ctypes.c_int32 * ISD_COPY_BITS),
        ("copy_nbr1", ctypes.c_uint64 * ISD_COPY_BITS),
        ("copy_jneg1", ctypes.c_uint64 * ISD_COPY_BITS),
        ("copy_nbr2", ctypes.c_uint64 * ISD_COPY_BITS),
        ("copy_jneg2", ctypes.c_uint64 * ISD_COPY_BITS),
        ("copy_table", ctypes.c_int32 * (1 << ISD_COPY_BITS)),
        ("e_mode", ctypes.c_uint32), ("e_parity", ctypes.c_uint32),
        ("odd_mask", ctypes.c_uint64),
        ("row_words", ctypes.c_uint32), ("e_words", ctypes.c_uint32),
        ("plane_words", ctypes.c_uint32), ("hist_words", ctypes.c_uint32),
        ("lane_mask", ctypes.c_uint64), ("lane_vec", ctypes.c_uint64 * 5),
        ("est_wavefronts", ctypes.c_double),
        ("pair_mode", ctypes.c_uint32), ("pair_degree", ctypes.c_int32 * 2),
        ("pair_words", ctypes.c_uint32 * 2), ("pair_both", ctypes.c_int32),
        ("base_words", ctypes.c_uint32),
        ("band_rows", ctypes.c_uint32), ("band_span", ctypes.c_uint32),
        ("est_per_config", ctypes.c_double),
    ]


class NativeError(RuntimeError):
    """A failure reported by the native engine (CUDA error, no device...)."""


_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return os.environ.get("ISD_LIBRARY", LIB)


def load():
    """Load (once) and return the ctypes handle; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not os.path.exists(path):
            raise ImportError(
                f"isingdos-b200 native library not found at {path}; build it "
                f"with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        u64, i32, dbl = ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        p_lat = ctypes.POINTER(Lattice)
        p_dbl = ctypes.POINTER(ctypes.c_double)
        vp = ctypes.c_void_p
        # (host buffers cross as plain addresses: ndarray.ctypes.data_as
        # costs ~4 us per call, .ctypes.data ~1 us)
        lib.isd_enumerate.argtypes = [p_lat, u64, u64, i32, i32, vp, p_dbl]
        lib.isd_enumerate_async.argtypes = [p_lat, u64, u64, i32, vp, i32, vp,
                                            ctypes.POINTER(ctypes.c_int)]
        lib.isd_thermo.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32,
                                   dbl, vp, i32, vp, i32, i32, vp, p_dbl]
        lib.isd_thermo_async.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32,
                                         dbl, vp, i32, vp, i32, vp, vp]
        lib.isd_mirror_async.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32,
                                         vp]
        lib.isd_plan.argtypes = [p_lat, u64, ctypes.POINTER(PlanInfo)]
        lib.isd_validate.argtypes = [p_lat]
        lib.isd_calibrate.argtypes = [i32, i32, p_dbl, p_dbl]
        lib.isd_sm_count.argtypes = [i32]
        lib.isd_last_error.restype = ctypes.c_char_p
        lib.isd_version.restype = ctypes.c_char_p
        lib.isd_kernel_info.restype = ctypes.c_char_p
        lib.isd_jit_check.argtypes = [p_lat, u64, ctypes.POINTER(ctypes.c_uint64)]
        lib.isd_jit_check.restype = ctypes.c_int
        lib.isd_band_items.argtypes = [
            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, vp,
            ctypes.c_uint32, dbl, vp, ctypes.c_uint32,
            ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int)]
        lib.isd_band_items.restype = ctypes.c_int
        lib.isd_launch_count.restype = ctypes.c_uint64
        lib.isd_set_knob.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
        lib.isd_set_knob.restype = ctypes.c_int
        lib.isd_clear_knobs.restype = ctypes.c_int
        lib.isd_enumerate_multi.argtypes = [p_lat, u64, u64, i32, vp, i32,
                                            vp, vp, p_dbl]
        lib.isd_enumerate_multi.restype = ctypes.c_int
        lib.isd_thermo_gather_async.argtypes = [
            vp, i32, vp, ctypes.c_uint32, ctypes.c_uint32, dbl, vp, i32, vp,
            i32, vp, vp]
        lib.isd_thermo_gather_async.restype = ctypes.c_int
        lib.isd_walk_plan.argtypes = [p_lat, u64, u64, i32,
                                      ctypes.POINTER(PlanInfo)]
        lib.isd_walk_plan.restype = ctypes.c_int
        lib.isd_set_walk_plan.argtypes = [p_lat, u64, u64,
                                          ctypes.POINTER(PlanInfo)]
        lib.isd_set_walk_plan.restype = ctypes.c_int
        lib.isd_band_costs.argtypes = [p_lat, ctypes.POINTER(PlanInfo), u64,
                                       ctypes.c_uint32, ctypes.c_uint32,
                                       ctypes.c_uint32, vp]
        lib.isd_band_costs.restype = ctypes.c_int
        lib.isd_band_slot_order.argtypes = [p_lat, ctypes.POINTER(PlanInfo),
                                            u64, ctypes.c_uint32, i32, vp]
        lib.isd_band_slot_order.restype = ctypes.c_int
        lib.isd_plan_range.argtypes = [p_lat, u64, u64, ctypes.POINTER(PlanInfo)]
        lib.isd_plan_range.restype = ctypes.c_int
        lib.isd_naive_enumerate.argtypes = [
            ctypes.c_uint32, vp, ctypes.c_uint32, vp, vp, i32, u64, u64, i32,
            vp]
        lib.isd_naive_enumerate.restype = ctypes.c_int
        lib.isd_enumerate_thermo.argtypes = [
            p_lat, u64, u64, i32, vp, i32, dbl, vp, i32, vp, i32, vp, vp, vp,
            p_dbl]
        lib.isd_enumerate_thermo.restype = ctypes.c_int
        lib.isd_set_cache_dirs.argtypes = [ctypes.c_char_p]
        lib.isd_set_cache_dirs.restype = ctypes.c_int
        lib.isd_build_id.restype = ctypes.c_char_p
        for name in ("isd_enumerate", "isd_enumerate_async", "isd_thermo",
                     "isd_thermo_async", "isd_plan", "isd_validate",
                     "isd_calibrate", "isd_device_count", "isd_sm_count",
                     "isd_abi_version", "isd_mirror_async"):
            getattr(lib, name).restype = ctypes.c_int
        if lib.isd_abi_version() != 2:
            raise ImportError("isingdos-b200 ABI version mismatch")
        lib.isd_set_cache_dirs(default_cache_dir().encode())
        _lib = lib
        return lib


def default_cache_dir() -> str:
    """Where tuned plans and NVRTC cubins persist between processes:
    $XDG_CACHE_HOME/isingdos_b200 (default ~/.cache/isingdos_b200)."""
    base = os.environ.get("XDG_CACHE_HOME") or os.path.join(
        os.path.expanduser("~"), ".cache")
    return os.path.join(base, "isingdos_b200")


def set_cache_dirs(dirs) -> None:
    """Set the engine's plan / cubin cache: a path, a list of paths (the
    first is written, the rest are read-only seeds), or None to disable."""
    if dirs is None:
        text = ""
    elif isinstance(dirs, str):
        text = dirs
    else:
        text = ":".join(dirs)
    check(load().isd_set_cache_dirs(text.encode()))


def build_id() -> str:
    return load().isd_build_id().decode()


def check(rc: int) -> None:
    if rc != 0:
        msg = load().isd_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise NativeError(f"isingdos-b200 native error {rc}: {msg}")


def set_knob(name: str, value=None) -> None:
    """Set (or with None unset) one tuning knob of the engine.

    Knobs force planning and launch choices (loop width, pairing mode,
    banded tables, autotuning, the JIT...) for the tests and tools/; the
    library never reads them from the environment (include/isingdos_b200.h).
    """
    v = None if value is None else str(value).encode()
    check(load().isd_set_knob(name.encode(), v))


def clear_knobs() -> None:
    load().isd_clear_knobs()


@contextlib.contextmanager
def knobs(**values):
    """Set knobs for the duration of a block: `with knobs(ISD_JIT=2): ...`."""
    for k, v in values.items():
        set_knob(k, v)
    try:
        yield
    finally:
        for k in values:
            set_knob(k, None)


def make_lattice(n_spins, n_bonds, classes) -> Lattice:
    """classes: iterable of (shift, bond_mask, jneg_mask)."""
    classes = list(classes)
    if not 1 <= len(classes) <= ISD_MAX_CLASSES:
        raise ValueError(f"{len(classes)} bond classes (1..{ISD_MAX_CLASSES})")
    lat = Lattice()
    lat.n_spins = n_spins
    lat.n_bonds = n_bonds
    lat.n_classes = len(classes)
    for i, (s, m, j) in enumerate(classes):
        lat.classes[i].shift = s
        lat.classes[i].bond_mask = m
        lat.classes[i].jneg_mask = j
    return lat


def _default_device() -> int:
    env = os.environ.get("ISD_DEVICE")
    if env:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


_device = None


def set_device(device: int) -> None:
    global _device
    _device = int(device)


def current_device() -> int:
    return _device if _device is not None else _default_device()


def device_count() -> int:
    return int(load().isd_device_count())


def enumerate_host(lat: Lattice, start: int, end: int, device=None,
                   algo: int = ALGO_AUTO):
    """Run the enumeration into a fresh host table; (uint64 table, device ms)."""
    lib = load()
    out = np.zeros((lat.n_spins + 1) * (lat.n_bonds + 1), dtype=np.uint64)
    ms = ctypes.c_double(0.0)
    dev = current_device() if device is None else device
    check(lib.isd_enumerate(ctypes.byref(lat), start, end, dev, algo,
                            out.ctypes.data,
                            ctypes.byref(ms)))
    return out.reshape(lat.n_spins + 1, lat.n_bonds + 1), ms.value


def enumerate_multi(lat: Lattice, start: int, end: int, devices,
                    algo: int = ALGO_AUTO):
    """Walk [start, end) as len(devices) shards, shard i on devices[i]
    (the reference's partition), tables combined on devices[0] by a peer
    gather kernel.  Returns (uint64 table, per-shard device ms, root ms)."""
    lib = load()
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    if devs.ndim != 1 or len(devs) < 1:
        raise ValueError("need at least one device")
    out = np.zeros((lat.n_spins + 1) * (lat.n_bonds + 1), dtype=np.uint64)
    shard_ms = np.zeros(len(devs), dtype=np.float64)
    total = ctypes.c_double(0.0)
    check(lib.isd_enumerate_multi(ctypes.byref(lat), start, end, len(devs),
                                  devs.ctypes.data, algo, out.ctypes.data,
                                  shard_ms.ctypes.data, ctypes.byref(total)))
    return (out.reshape(lat.n_spins + 1, lat.n_bonds + 1), shard_ms.tolist(),
            total.value)


def enumerate_thermo(lat: Lattice, start: int, end: int, devices,
                     scale: float, fields, temps, algo: int = ALGO_AUTO):
    """Walk + combine + thermodynamic grid in one engine call
    (isd_enumerate_thermo).  Returns (uint64 table, float64 [F, T, 7],
    per-shard device ms, root ms)."""
    lib = load()
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    f = np.ascontiguousarray(fields, dtype=np.float64)
    t = np.ascontiguousarray(temps, dtype=np.float64)
    out = np.zeros((lat.n_spins + 1) * (lat.n_bonds + 1), dtype=np.uint64)
    grid = np.empty((len(f), len(t), ISD_THERMO_FIELDS), dtype=np.float64)
    shard_ms = np.zeros(len(devs), dtype=np.float64)
    total = ctypes.c_double(0.0)
    check(lib.isd_enumerate_thermo(
        ctypes.byref(lat), start, end, len(devs), devs.ctypes.data, algo,
        float(scale), f.ctypes.data, len(f), t.ctypes.data, len(t),
        out.ctypes.data, grid.ctypes.data, shard_ms.ctypes.data,
        ctypes.byref(total)))
    return (out.reshape(lat.n_spins + 1, lat.n_bonds + 1), grid,
            shard_ms.tolist(), total.value)


def thermo_gather_device(table_ptrs, sum_ptr, n_spins, n_bonds, scale,
                         fields_ptr, n_fields, temps_ptr, n_temps, out_ptr,
                         stream_ptr) -> int:
    """Fused sum of several device tables + K2 (isd_thermo_gather_async);
    returns the kernels launched."""
    lib = load()
    ptrs = (ctypes.c_void_p * len(table_ptrs))(*table_ptrs)
    check(lib.isd_thermo_gather_async(
        ptrs, len(table_ptrs), ctypes.c_void_p(sum_ptr or None), n_spins,
        n_bonds, float(scale), ctypes.c_void_p(fields_ptr or None), n_fields,
        ctypes.c_void_p(temps_ptr or None), n_temps,
        ctypes.c_void_p(out_ptr or None), ctypes.c_void_p(stream_ptr)))
    gather = 1 if len(table_ptrs) > 1 or sum_ptr else 0  # K4
    return gather + (1 if n_fields * n_temps > 0 else 0)   # + K2


def naive_enumerate(bit_of_slot, bonds, coupling_sign: int, start: int,
                    end: int, device=None):
    """The naive engine (K5): spins decoded per slot, E summed over the
    explicit bond list `bonds` = [(slot_i, slot_j, sign)]; uint64 table."""
    lib = load()
    pos = np.ascontiguousarray(bit_of_slot, dtype=np.uint32)
    n = len(pos)
    slots = np.ascontiguousarray([(i, j) for i, j, _ in bonds],
                                 dtype=np.uint32).reshape(-1)
    signs = np.ascontiguousarray([s for _, _, s in bonds], dtype=np.int32)
    out = np.zeros((n + 1) * (len(bonds) + 1), dtype=np.uint64)
    dev = current_device() if device is None else device
    check(lib.isd_naive_enumerate(
        n, pos.ctypes.data, len(bonds), slots.ctypes.data if len(bonds) else None,
        signs.ctypes.data if len(bonds) else None, int(coupling_sign), start,
        end, dev, out.ctypes.data))
    return out.reshape(n + 1, len(bonds) + 1)


def enumerate_device(lat: Lattice, start: int, end: int, counts_ptr: int,
                     stream_ptr: int, accumulate: bool = False,
                     algo: int = ALGO_AUTO) -> int:
    """Enqueue on a device table (raw pointer) and stream; returns launches."""
    lib = load()
    nl = ctypes.c_int(0)
    check(lib.isd_enumerate_async(ctypes.byref(lat), start, end, algo,
                                  ctypes.c_void_p(counts_ptr), int(accumulate),
                                  ctypes.c_void_p(stream_ptr),
                                  ctypes.byref(nl)))
    return nl.value


def thermo_host(counts, n_spins, n_bonds, scale, fields, temps, device=None):
    """fp64 thermodynamics of a host table; returns (array[F, T, 7], ms)."""
    lib = load()
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    f = np.ascontiguousarray(fields, dtype=np.float64)
    t = np.ascontiguousarray(temps, dtype=np.float64)
    out = np.empty((len(f), len(t), ISD_THERMO_FIELDS), dtype=np.float64)
    ms = ctypes.c_double(0.0)
    dev = current_device() if device is None else device
    check(lib.isd_thermo(c.ctypes.data, n_spins, n_bonds, float(scale),
                         f.ctypes.data, len(f), t.ctypes.data, len(t), dev,
                         out.ctypes.data, ctypes.byref(ms)))
    return out, ms.value


def thermo_device(counts_ptr, n_spins, n_bonds, scale, fields_ptr, n_fields,
                  temps_ptr, n_temps, out_ptr, stream_ptr) -> int:
    lib = load()
    check(lib.isd_thermo_async(ctypes.c_void_p(counts_ptr), n_spins, n_bonds,
                               float(scale), ctypes.c_void_p(fields_ptr),
                               n_fields, ctypes.c_void_p(temps_ptr), n_temps,
                               ctypes.c_void_p(out_ptr),
                               ctypes.c_void_p(stream_ptr)))
    return 1 if n_fields * n_temps > 0 else 0  # K2


def plan(lat: Lattice, n_configs_hint: int) -> tuple:
    """Host-side hoisted-kernel plan (no GPU needed): (usable, PlanInfo)."""
    lib = load()
    info = PlanInfo()
    rc = lib.isd_plan(ctypes.byref(lat), n_configs_hint, ctypes.byref(info))
    if rc < 0:
        check(rc)
    return rc == 0, info


def walk_plan(lat: Lattice, start: int, end: int, device=None) -> tuple:
    """The plan a walk of [start, end) runs with on `device` (autotuned for
    walks of >= 2^33 configurations): (usable, PlanInfo)."""
    lib = load()
    info = PlanInfo()
    dev = current_device() if device is None else device
    rc = lib.isd_walk_plan(ctypes.byref(lat), start, end, dev,
                           ctypes.byref(info))
    if rc < 0:
        check(rc)
    return rc == 0, info


def set_walk_plan(lat: Lattice, start: int, end: int, info: PlanInfo) -> None:
    """Use `info` for walks of [start, end)'s size and top bits (tools)."""
    check(load().isd_set_walk_plan(ctypes.byref(lat), start, end,
                                   ctypes.byref(info)))


def plan_fingerprint(info: PlanInfo) -> str:
    """Short stable digest of a plan (to compare plans across processes)."""
    import hashlib
    return hashlib.sha256(bytes(info)).hexdigest()[:16]


def plan_range(lat: Lattice, start: int, end: int) -> tuple:
    """Host model plan of a walk of [start, end) (top bits of an aligned
    power-of-two range fixed, as the walk holds them): (usable, PlanInfo)."""
    info = PlanInfo()
    rc = load().isd_plan_range(ctypes.byref(lat), start, end, ctypes.byref(info))
    if rc < 0:
        check(rc)
    return rc == 0, info


def validate(lat: Lattice) -> None:
    check(load().isd_validate(ctypes.byref(lat)))


def calibrate(which: int, device=None):
    lib = load()
    lanes = ctypes.c_double(0.0)
    mhz = ctypes.c_double(0.0)
    dev = current_device() if device is None else device
    check(lib.isd_calibrate(dev, which, ctypes.byref(lanes), ctypes.byref(mhz)))
    return lanes.value, mhz.value


def launch_count() -> int:
    return int(load().isd_launch_count())


def sm_count(device=None) -> int:
    dev = current_device() if device is None else device
    v = load().isd_sm_count(dev)
    if v < 0:
        check(v)
    return v


def kernel_info() -> str:
    """Kernel path of the last enumeration on this thread."""
    return load().isd_kernel_info().decode()


def jit_check(lat: Lattice, n_configs_hint: int) -> int:
    """NVRTC-compile the lattice's specialised kernel (no GPU); cubin bytes."""
    n = ctypes.c_uint64(0)
    check(load().isd_jit_check(ctypes.byref(lat), n_configs_hint,
                               ctypes.byref(n)))
    return n.value


def band_costs(lat: Lattice, info: PlanInfo, run_begin: int, run_bits: int,
               n_seg: int, samples: int = 64):
    """The host model's cost curve of a banded launch (no GPU; tools)."""
    out = np.zeros(n_seg, dtype=np.float64)
    n = load().isd_band_costs(ctypes.byref(lat), ctypes.byref(info),
                              run_begin, run_bits, n_seg, samples,
                              out.ctypes.data)
    if n < 0:
        check(n)
    return out[:n]


def band_slot_order(lat: Lattice, info: PlanInfo, run_begin: int,
                    run_bits: int, reorder: bool = True):
    """Run bit of every slot bit of a banded launch (no GPU; tools/tests)."""
    out = np.zeros(24, dtype=np.uint8)
    n = load().isd_band_slot_order(ctypes.byref(lat), ctypes.byref(info),
                                   run_begin, run_bits, 1 if reorder else 0,
                                   out.ctypes.data)
    if n < 0:
        check(n)
    return out[:n]


def band_items(free_bits: int, n_target: int, span: int, seg_cost=None,
               flush_units: float = 20.0):
    """The host's work-item split of a banded launch (no GPU; for tests):
    (array[n, 3] of (g0, g1, q0), exact)."""
    lib = load()
    w = (np.ascontiguousarray(seg_cost, dtype=np.float64)
         if seg_cost is not None else np.zeros(0))
    cap = 4 * n_target + 64
    out = np.zeros(3 * cap, dtype=np.uint64)
    n = ctypes.c_uint32(0)
    ex = ctypes.c_int(0)
    check(lib.isd_band_items(free_bits, n_target, span,
                             w.ctypes.data if len(w) else None, len(w),
                             float(flush_units), out.ctypes.data, cap,
                             ctypes.byref(n), ctypes.byref(ex)))
    return out[:3 * n.value].reshape(-1, 3).astype(np.int64), bool(ex.value)

