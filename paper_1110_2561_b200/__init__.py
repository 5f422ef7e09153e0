"""isingdos-b200: exact density of states of finite Ising lattices on B200.

A B200-native engine behind the public API of the reference package
`isingdos` (/root/reference/pkg/src/isingdos/__init__.py:10-38) for its hot
path: lattice construction, exhaustive sharded enumeration into the exact
integer table g(M, E), verification, and fp64 thermodynamics Z(h, T).
Enumeration (K1) and thermodynamics (K2) are hand-written sm_100a kernels
behind the C ABI in include/isingdos_b200.h; multi-GPU runs shard the index
space by its top bits and combine the per-GPU tables with one NCCL reduce
(`paper_1110_2561_b200.distributed`).
"""

from ._native import NativeError, current_device, set_device
from .crosscheck import (
    ORACLE_MAX_SPINS,
    brute_force_log_z,
    decode_spins,
    oracle_energy,
    oracle_full_dos,
    oracle_magnetization,
)
from .bench import (
    BenchRecord,
    ResultMismatchError,
    emit_scaling_report,
    parse_scaling_report,
    run_bench,
)
from .dosio import (
    DosFileError,
    format_dos_csv,
    format_dos_json,
    parse_dos,
    read_dos,
    write_dos,
)
from .enumeration import (
    DEFAULT_BATCH,
    DoSHistogram,
    Shard,
    VerificationReport,
    available_parallelism,
    enumerate_shard,
    full_dos,
    full_dos_timed,
    gpu_count,
    make_shards,
    merge,
    verify_dos,
)
from .lattice import (
    MAX_ROWS,
    MAX_SPINS,
    TABLE_ROWS_CAP,
    Configuration,
    KernelTables,
    LatticeSpec,
    aligned_column_bonds,
    aligned_row_bonds,
    build_tables,
    circular_shift,
    decode_config,
    encode_words,
    popcount,
    random_bond_signs,
    spin_excess,
    total_energy,
    unsatisfied_bonds,
)
from .thermo import (
    ThermoPoint,
    dos_thermo,
    partition_point,
    temperature_grid,
    thermo_grid,
    thermo_sweep,
)

__version__ = "0.1.0"

__all__ = [
    "BenchRecord", "DosFileError", "ResultMismatchError",
    "emit_scaling_report", "format_dos_csv", "format_dos_json", "parse_dos",
    "parse_scaling_report", "read_dos", "run_bench", "write_dos",
    "Configuration", "DEFAULT_BATCH", "DoSHistogram", "KernelTables",
    "LatticeSpec", "MAX_ROWS", "MAX_SPINS", "NativeError", "Shard",
    "TABLE_ROWS_CAP", "ThermoPoint", "VerificationReport",
    "aligned_column_bonds", "aligned_row_bonds", "available_parallelism",
    "build_tables", "circular_shift", "current_device", "decode_config",
    "encode_words", "enumerate_shard", "full_dos", "full_dos_timed",
    "gpu_count", "make_shards", "merge", "partition_point", "popcount",
    "random_bond_signs", "set_device", "spin_excess", "temperature_grid",
    "thermo_grid", "thermo_sweep", "dos_thermo", "total_energy", "unsatisfied_bonds",
    "verify_dos", "ORACLE_MAX_SPINS", "brute_force_log_z", "decode_spins",
    "oracle_energy", "oracle_full_dos", "oracle_magnetization",
]
