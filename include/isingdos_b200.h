/*
 * isingdos_b200.h — C ABI of the B200 exact-enumeration engine.
 *
 * The reference (`isingdos`, /root/reference/pkg/src/isingdos) is pure
 * Python/numpy and has no FFI; its hot path is
 *
 *   enumerate_shard(spec, tables, shard, batch_size)   enumeration.py:208-235
 *     -> _classify_batch(...)                          enumeration.py:167-205
 *     -> np.bincount accumulate                        enumeration.py:232-234
 *   full_dos_timed / full_dos (Pool driver + root sum) enumeration.py:365-396
 *   partition_point / thermo_sweep                     thermo.py:46-100
 *
 * Each entry point below replaces one of those loops; the call a
 * maintainer would add to the reference (ctypes) is shown in
 * INTEGRATION.md.  Conventions:
 *   - plain pointers and sizes only; no torch / CUDA runtime types;
 *   - every function returns 0 on success and a negative ISD_E* code on
 *     failure, with a message in isd_last_error() (thread-local);
 *   - host output buffers are caller-owned and fully overwritten;
 *   - `stream` arguments are cudaStream_t passed as void* (NULL = legacy
 *     default stream of the current device);
 *   - the library never keeps caller pointers.
 *
 * Lattice description.  The reference's geometry (LatticeSpec,
 * lattice.py:34-119, and oracle.bond_pairs, oracle.py:40-58) is compiled on
 * the host into at most ISD_MAX_CLASSES "bond classes".  A class is a shift
 * s and two N-bit masks: bit i of bond_mask says bond (i, i+s) exists, bit i
 * of jneg_mask says that bond has negative sign (it is unsatisfied when the
 * two spins are ALIGNED).  For configuration index x (bit i = spin of site i,
 * 1 = up; lattice.py:1-13):
 *
 *   m_idx = popcount(x)                                   (= (M+N)/2)
 *   e_idx = sum_c popcount(((x ^ (x >> s_c)) ^ jneg_c) & bond_c)
 *
 * e_idx counts unsatisfied bonds, E = |J| (2 e_idx - B): identical to the
 * reference's column index (enumeration.py:95-121, 232-233).  Counts are
 * written as a dense row-major uint64 table counts[m_idx][e_idx] of shape
 * (N+1) x (B+1) — the reference's DoSHistogram.counts layout.
 */
#ifndef ISINGDOS_B200_H
#define ISINGDOS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISD_ABI_VERSION 2
#define ISD_MAX_CLASSES 8
#define ISD_MAX_SPINS 40   /* lattice.py:24 MAX_SPINS */

/* error codes */
#define ISD_OK 0
#define ISD_EINVAL (-1)   /* bad argument (range, lattice, sizes)        */
#define ISD_ECUDA (-2)    /* CUDA runtime failure                        */
#define ISD_ENODEV (-3)   /* no CUDA device / bad device ordinal          */
#define ISD_ENOMEM (-4)   /* device allocation failed                     */

/* enumeration algorithms (isd_enumerate*.algo) */
#define ISD_ALGO_AUTO 0       /* hoisted kernel for the aligned body, canonical head/tail */
#define ISD_ALGO_CANONICAL 1  /* one full class-mask evaluation per configuration */
#define ISD_ALGO_HOISTED 2    /* same as AUTO; errors if the lattice is too small */
/* OR-able flag: walk only the configurations with the top spin down and
 * complete the table with g(M, E) = h(M, E) + h(-M, E) (global spin flip
 * preserves E for any couplings at zero field).  Only for full walks
 * [0, 2^N); halves the enumerated configurations (reported separately). */
#define ISD_FLAG_FLIP_SYMMETRY 0x100

typedef struct isd_bond_class {
  uint32_t shift;     /* partner offset s, 1 <= s < N                    */
  uint32_t reserved;  /* must be 0                                       */
  uint64_t bond_mask; /* bit i: bond (i, i+s) exists (i+s < N)           */
  uint64_t jneg_mask; /* bit i: that bond is antiferro (subset of bond)  */
} isd_bond_class;

typedef struct isd_lattice {
  uint32_t n_spins;   /* N, 1..40                                        */
  uint32_t n_bonds;   /* B = sum_c popcount(bond_mask_c)                 */
  uint32_t n_classes; /* 1..ISD_MAX_CLASSES                              */
  uint32_t reserved;  /* must be 0                                       */
  isd_bond_class classes[ISD_MAX_CLASSES];
} isd_lattice;

/* ---- enumeration (replaces enumerate_shard, enumeration.py:208-235) ---- */

/* Host-buffer call: walks [start, end) on `device`, writes the exact
 * (N+1)*(B+1) table to counts_host (zeroed first).  Synchronous.  Returns the
 * device time of the kernels in *device_ms when non-NULL. */
int isd_enumerate(const isd_lattice* lat, uint64_t start, uint64_t end,
                  int device, int algo, uint64_t* counts_host,
                  double* device_ms);

/* Device-buffer call: accumulates (accumulate=1) or overwrites
 * (accumulate=0) the table at counts_dev (device memory of the current
 * device) on `stream`.  Asynchronous; *launches receives the number of
 * kernels enqueued when non-NULL. */
int isd_enumerate_async(const isd_lattice* lat, uint64_t start, uint64_t end,
                        int algo, uint64_t* counts_dev, int accumulate,
                        void* stream, int* launches);

/* Multi-device walk (replaces full_dos_timed's Pool of shard workers and
 * its root-side sum, enumeration.py:365-390).  Splits [start, end) into
 * n_shards contiguous shards with the reference's partition (make_shards,
 * enumeration.py:44-63; for n_shards = 2^k over an aligned power-of-two
 * range: the top k index bits) and walks shard i on device devs[i].  A
 * device may be listed several times: its shards then run one after another
 * on its stream (so on one GPU every shard of a P-way split is timed on its
 * own).  The tables are combined on the device: the root devs[0] reads every
 * device's table over NVLink peer access (or a device-to-device copy where
 * peer access is unavailable) in one kernel.  Writes the exact table to
 * counts_host, shard i's device time to shard_ms[i] (NULL: not wanted) and
 * the root's span — from its start event, which every device waits on, to
 * the combined table — to *total_ms.  ISD_FLAG_FLIP_SYMMETRY: the shards
 * split the top-spin-down half of the full range and the root completes
 * the table.  Synchronous. */
int isd_enumerate_multi(const isd_lattice* lat, uint64_t start, uint64_t end,
                        int n_shards, const int* devs, int algo,
                        uint64_t* counts_host, double* shard_ms,
                        double* total_ms);

/* The naive cross-check engine (replaces oracle_full_dos's per-index loop,
 * oracle.py:71-91): per configuration, decode every spin S = +-1 from bit
 * bit_of_slot[s] of the index, M = sum of spins, and E / |J| =
 * -sign(J) * sum_b bond_sign[b] S_i S_j over the explicit bond list
 * (bond_slots[2b], bond_slots[2b + 1]) — one thread per configuration,
 * nothing shared with the enumeration kernels or the bond-class
 * descriptor.  Writes the (N+1) x (B+1) table of [start, end) like
 * isd_enumerate.  Synchronous. */
int isd_naive_enumerate(uint32_t n_spins, const uint32_t* bit_of_slot,
                        uint32_t n_bonds, const uint32_t* bond_slots,
                        const int32_t* bond_sign, int coupling_sign,
                        uint64_t start, uint64_t end, int device,
                        uint64_t* counts_host);

/* The whole pipeline in one call: isd_enumerate_multi, then on the root
 * the thermodynamic grid of the combined table (as isd_thermo) — host grid
 * in, host table and results out, one synchronisation.  The table of a
 * full walk [0, 2^N) is what the grid is evaluated from; the caller checks
 * completeness (thermo.py:59-63).  out_host: ISD_THERMO_FIELDS doubles per
 * (field, temperature) point, field-major. */
int isd_enumerate_thermo(const isd_lattice* lat, uint64_t start, uint64_t end,
                         int n_shards, const int* devs, int algo,
                         double energy_scale, const double* fields,
                         int n_fields, const double* temps, int n_temps,
                         uint64_t* counts_host, double* out_host,
                         double* shard_ms, double* total_ms);

/* In-place completion of a half walk: counts[m][e] += counts[N-m][e]
 * pairwise (rows m and N-m both become the sum).  Device buffer, async. */
int isd_mirror_async(uint64_t* counts_dev, uint32_t n_spins, uint32_t n_bonds,
                     void* stream);

/* ---- thermodynamics (replaces partition_point/thermo_sweep, thermo.py:46-100)
 * For every (field f, temperature t) pair, in field-major order
 * (index = f*n_temps + t), writes ISD_THERMO_FIELDS doubles:
 *   [log_z, free_energy, internal_energy, specific_heat,
 *    mean_magnetization, susceptibility, mean_abs_magnetization]
 * following thermo.py:65-77 (max-shifted log-sum-exp over occupied cells,
 * central second moments).  energy_scale = |J|.  Temperatures must be > 0
 * (validated by the caller, thermo.py:56-58). */
#define ISD_THERMO_FIELDS 7

int isd_thermo(const uint64_t* counts_host, uint32_t n_spins, uint32_t n_bonds,
               double energy_scale, const double* fields, int n_fields,
               const double* temps, int n_temps, int device, double* out_host,
               double* device_ms);

int isd_thermo_async(const uint64_t* counts_dev, uint32_t n_spins,
                     uint32_t n_bonds, double energy_scale,
                     const double* fields_dev, int n_fields,
                     const double* temps_dev, int n_temps, double* out_dev,
                     void* stream);

/* The fused combine + thermodynamics of a multi-GPU step: the tables
 * tables_dev[0 .. n_tables) (device pointers readable from the current
 * device: its own, peer-mapped NVLink memory, or CUDA IPC mappings of other
 * processes' tables) are summed inside K2's compaction kernel, the sum is
 * written to sum_dev (may be NULL when a grid is given) and the grid is
 * evaluated from it, as isd_thermo_async.  With an empty grid only the sum
 * is formed (one gather kernel).  n_tables <= 32.  Asynchronous on
 * `stream`. */
int isd_thermo_gather_async(const uint64_t* const* tables_dev, int n_tables,
                            uint64_t* sum_dev, uint32_t n_spins,
                            uint32_t n_bonds, double energy_scale,
                            const double* fields_dev, int n_fields,
                            const double* temps_dev, int n_temps,
                            double* out_dev, void* stream);

/* ---- host-side plan (no GPU needed; used by the CPU tests) ----------- */

/* The hoisted kernel's decomposition of the lattice.
 * The low k index bits are split into u "copy" sites (unrolled in
 * registers) and l loop sites (the thread's loop counter, enumerated as the
 * subsets of loop_mask); bits [k, N) are the per-thread run prefix. */
#define ISD_COPY_BITS 7
typedef struct isd_plan_info {
  uint32_t u, l, k;          /* k = u + l                               */
  uint32_t stride;           /* B + 1                                   */
  uint64_t run_mask_above_k; /* bits [k, N)                             */
  uint64_t loop_mask;        /* the l loop sites (bits of [0, k))        */
  int32_t  copy_site[ISD_COPY_BITS];     /* site of copy bit t            */
  int32_t  copy_degree[ISD_COPY_BITS];   /* bonds to non-copy sites       */
  uint64_t copy_nbr1[ISD_COPY_BITS];     /* non-copy partner masks        */
  uint64_t copy_jneg1[ISD_COPY_BITS];    /* partner sign masks            */
  uint64_t copy_nbr2[ISD_COPY_BITS];     /* second copy (double bonds)    */
  uint64_t copy_jneg2[ISD_COPY_BITS];
  int32_t  copy_table[1 << ISD_COPY_BITS]; /* popc(c)(B+1) + copy-copy unsat */
  /* Shared-histogram layout.  e_mode 0: word = m*row_words + e*e_words.
   * e_mode 1 (every copy site has even degree): e_idx has the parity
   * par(x) = (popc(x & odd_mask) + e_parity) & 1, constant over the 128
   * copies of a group, and word = m*row_words + ((e - par)/2)*e_words +
   * par*plane_words (two half-size parity planes; one plane when odd_mask
   * is 0).  Strides and the lane placement minimise bank conflicts. */
  uint32_t e_mode;
  uint32_t e_parity;
  uint64_t odd_mask;         /* sites of odd degree                     */
  uint32_t row_words;
  uint32_t e_words;
  uint32_t plane_words;
  uint32_t hist_words;       /* words spanned by one histogram          */
  uint64_t lane_mask;        /* the 5 pivot run bits of the lanes       */
  uint64_t lane_vec[5];      /* lane bit i flips the run bits lane_vec[i]
                                (its pivot, plus an optional adjacent
                                site: a "domino"); lane L's run is the
                                slot's run XOR the vectors of L's bits  */
  double   est_wavefronts;   /* predicted smem wavefronts per warp RED  */
  /* Paired copies.  pair_mode 1: copy bit 6's site q is not a register
   * copy of its own; one RED counts the configuration with q down AND its
   * partner with q up: it lands in pattern plane p = (bonds of q left
   * unsatisfied while q is down), word = base word + p*pair_words[0], and
   * the flush credits the partner to (m + 1, e + pair_degree[0] - 2p).
   * pair_mode 2 pairs copy bit 5 the same way on top (index 1 of the
   * arrays): one RED counts four configurations; the one with both sites
   * up lands at (m + 2, e + D0 - 2p0 + D1 - 2p1 + pair_both).  Each pairing
   * halves the shared-memory REDs per configuration and multiplies the
   * histogram by D + 1 planes of base_words words.
   * pair_mode 3: copy bits 4, 5, 6 are a cluster of three like sites
   * (equal degree, each pair joined by the same w = 0 or 1 bonds of one
   * sign, no bond to the unpaired copy sites): one RED counts the
   * cluster's 8 configurations, in the plane of the multiset {a, b, c} of
   * the three sites' unsatisfied external bonds (each 0..R, R = D - 2w):
   * word = base word + tri(a, b, c)*pair_words[0], (R+1)(R+2)(R+3)/6
   * planes; the flush credits the subset U flipped up to
   * (m + |U|, e + sum_U (R - 2 n_i) + [|U| = 1 or 2] pair_both). */
  uint32_t pair_mode;        /* 0, 1, 2 or 3                            */
  int32_t  pair_degree[2];   /* degree D of the paired sites (bit 6, 5);
                                mode 3: {R, w}                          */
  uint32_t pair_words[2];    /* pattern-plane strides (bit 6, bit 5);
                                mode 3: {plane stride, plane count}     */
  int32_t  pair_both;        /* mode 2: e change of flipping both sites
                                beyond the sum of the single flips;
                                mode 3: 2w(1 - 2 neg), the internal-bond
                                term of one or two cluster sites up     */
  uint32_t base_words;       /* words of the unpaired layout            */
  /* Banded tables (band_rows > 0, pairing modes 2 and 3): the table holds
   * band_rows rows of m relative to a base row, and a launch is split into
   * work items of run slots ordered by popcount, each item's runs spanning
   * at most band_span + 5 + l + u - pair_mode rows — so a table that could
   * not hold all N + 1 rows fits shared memory.  Lanes are then single
   * run sites (lane_vec[i] == pivot i). */
  uint32_t band_rows;
  uint32_t band_span;
  double   est_per_config;   /* est_wavefronts / configurations per RED */
} isd_plan_info;

int isd_plan(const isd_lattice* lat, uint64_t n_configs_hint,
             isd_plan_info* out);

/* The plan a walk of [start, end) on `device` actually runs with: the
 * host model's for small walks, the autotuned one (from memory, the disk
 * cache, or tuned now) for walks of >= 2^33 configurations.  Returns 0, or
 * > 0 when the lattice is too small for the hoisted kernel. */
int isd_walk_plan(const isd_lattice* lat, uint64_t start, uint64_t end,
                  int device, isd_plan_info* out);

/* Install `plan` as the plan of walks of [start, end)'s size and top
 * bits in this process (replacing the tuned one; not written to the disk
 * cache).  For tools and tests that time one plan on several ranges; the
 * plan must come from isd_plan / isd_walk_plan of the same lattice. */
int isd_set_walk_plan(const isd_lattice* lat, uint64_t start, uint64_t end,
                      const isd_plan_info* plan);

/* The host model's plan for a walk of [start, end) (no GPU): as isd_plan,
 * but an aligned power-of-two range is planned with its top bits fixed, as
 * the walk itself is.  The GPU autotuner starts from this model. */
int isd_plan_range(const isd_lattice* lat, uint64_t start, uint64_t end,
                   isd_plan_info* out);

/* Generate and NVRTC-compile the lattice's specialised k1 kernel without
 * loading it (no GPU needed); *cubin_bytes = its size.  For tests. */
int isd_jit_check(const isd_lattice* lat, uint64_t n_configs_hint,
                  uint64_t* cubin_bytes);

/* Validate a lattice descriptor without touching a GPU. */
int isd_validate(const isd_lattice* lat);

/* The host's work-item split of a banded launch over 2^free_bits slots (no
 * GPU needed; for tests): n_target items of equal cost under the per-slot
 * costs seg_cost[0 .. n_seg) (the slots cut into n_seg equal segments in
 * popcount order; n_seg = 0: equal costs), each spanning at most span + 1
 * popcount classes, plus the small items of the extreme classes.  Writes
 * (g0, g1, q0) per item to out (3 x max_items) and the count to *n_items;
 * *exact = 1 when item b is block b's first item. */
int isd_band_items(uint32_t free_bits, uint32_t n_target, uint32_t span,
                   const double* seg_cost, uint32_t n_seg, double flush_units,
                   uint64_t* out, uint32_t max_items, uint32_t* n_items,
                   int* exact);

/* The host model's per-segment cost of a banded launch (no GPU; tools and
 * tests): the 2^F slots of `run_bits` run bits from run_begin, in popcount
 * order, cut into n_seg segments; out[s] = expected shared wavefronts per
 * warp RED in segment s (`samples` sampled REDs).  Returns the segment
 * count written (<= n_seg) or a negative error. */
int isd_band_costs(const isd_lattice* lat, const isd_plan_info* plan,
                   uint64_t run_begin, uint32_t run_bits, uint32_t n_seg,
                   uint32_t samples, double* out);

/* The order of a banded launch's slot bits (no GPU; tools and tests): the
 * F = run_bits - 5 run bits that are not lane pivots, as pos_out[i] = the
 * run bit that bit i of a slot's popcount-ordered value lands on.  The run
 * sites that decide whether an item's table is cheaper with ascending or
 * descending rows take the most significant slot bits (reorder != 0), so
 * the slots of a work item agree on them; reorder == 0 gives the natural
 * order.  Returns F or a negative error. */
int isd_band_slot_order(const isd_lattice* lat, const isd_plan_info* plan,
                        uint64_t run_begin, uint32_t run_bits, int reorder,
                        uint8_t* pos_out);

/* ---- calibration microbenchmarks (K0) -------------------------------- */
/* which: 0 = POPC, 1 = LOP3, 2 = IADD3, 3 = RED.shared spread,
 *        4 = RED.shared realistic bins, 5 = IMAD, 6 = SHF, 7 = RED.shared
 *        all lanes on one word, 8 = lane pairs per word (16 banks),
 *        9 = 4 words in one bank, 10 = 8 words x 4 lanes, distinct banks,
 *        11 = all lanes one word with values 1 / 65536 (16-bit halves),
 *        12 = lane pairs per word with values 1 / 65536.  Writes lanes per clock
 *        per SM to *lanes_per_clk_sm and the SM clock seen (MHz). */
int isd_calibrate(int device, int which, double* lanes_per_clk_sm,
                  double* sm_mhz);

/* ---- tuning knobs ------------------------------------------------------
 * Process-wide overrides of planning and launch choices (loop width,
 * pairing mode, banded tables, autotuning, the JIT, ...), for the tests and
 * the experiment scripts.  The library never reads the environment: a knob
 * changes behaviour only when set here.  value NULL or "" unsets it; an
 * unknown name is ISD_EINVAL.  Plans are cached per knob set. */
int isd_set_knob(const char* name, const char* value);
int isd_clear_knobs(void);

/* ---- on-disk cache ------------------------------------------------------
 * Autotuned plans (walks of >= 2^33 configurations), band cost curves and
 * NVRTC cubins are kept in a directory cache so that a new process skips
 * the layout model, the GPU autotune and the compiles (and runs the same
 * plan as the process that tuned it).  `dirs` is a ':'-separated list: the
 * first directory is written (created if missing), the rest are read-only
 * seeds.  NULL or "" disables the cache (the default).  Entries are keyed
 * by isd_build_id(), the device name and SM count. */
int isd_set_cache_dirs(const char* dirs);
const char* isd_build_id(void);

/* ---- misc ------------------------------------------------------------ */
int isd_device_count(void);
int isd_sm_count(int device);
const char* isd_last_error(void);
/* Kernel path of the last enumeration on this thread: "k1_hoisted_jit"
 * (per-lattice NVRTC specialisation, walks >= 2^33), "k1_hoisted_aot",
 * "k1_canonical" (or an AOT note saying why the JIT was unavailable). */
const char* isd_kernel_info(void);
const char* isd_version(void);
int isd_abi_version(void);
/* Kernels launched by this process since load (all entry points). */
uint64_t isd_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* ISINGDOS_B200_H */
