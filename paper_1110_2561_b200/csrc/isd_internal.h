// Internal declarations shared by the host plan compiler, the kernels and the
// C ABI.  Nothing here is exported.
#pragma once

#include <cstdint>
#include <cstddef>
#include <string>
#include <vector>

#include "isingdos_b200.h"

#include <nvtx3/nvToolsExt.h>

namespace isd {

// NVTX range for the host phases (plan, autotune, NVRTC, prepare / issue of
// a walk): visible in nsys / ncu timelines, free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kCopyBits = ISD_COPY_BITS;   // u: sites unrolled in registers
// most loop sites the NVRTC kernel walks in Gray order (HoistParams.gray)
constexpr int kMaxGray = 5;
constexpr int kDefaultGray = 2;
constexpr int kCopies = 1 << kCopyBits;    // 128 configurations per group
static_assert(ISD_COPY_BITS == 7, "k1_hoisted emits 32 x 4 copies");
constexpr int kTreeBits = 5;               // copies emitted as a 32-leaf tree
                                           // plus outer bits 5..u-1
constexpr int kMaxClasses = ISD_MAX_CLASSES;
constexpr int kThreads = 512;              // threads per enumeration block
constexpr int kWideThreads = 1024;         // ... when only one block fits an
                                           // SM (large paired histograms)

// Parameters of the canonical kernel: one full class-mask evaluation per
// configuration (the formulation of enumeration.py:167-205 on bit masks).
struct CanonParams {
  uint64_t start, end;      // [start, end) configuration indices
  uint32_t n_classes;
  uint32_t stride;          // B + 1 (row length of the table)
  uint32_t nbins;           // (N+1)(B+1)
  uint32_t hist_words;      // words per shared histogram (padded)
  uint32_t n_hist;          // shared histograms per block
  uint32_t n_spins;         // N (selects the 32- or 64-bit index path)
  uint32_t shift[kMaxClasses];
  uint64_t mask[kMaxClasses];
  uint64_t jneg[kMaxClasses];
};

// Parameters of the hoisted kernel.  A "run" is 2^k
// consecutive indices: bits [k, N) are fixed per thread; inside [0, k) the
// loop sites (loop_mask) take every subset in the thread's loop and the 7
// copy sites are 128 register copies.
struct HoistParams {
  uint64_t run_begin, run_end;   // run indices (index = run << k)
  uint64_t above_k;              // bits [k, N)
  uint64_t odd_mask;             // odd-degree sites (parity planes)
  uint32_t loop_mask;            // loop sites
  uint32_t k, l;
  uint32_t n_classes;
  uint32_t stride;               // B + 1
  uint32_t nbins;
  uint32_t hist_words;           // words per shared histogram (padded)
  uint32_t n_hist;
  uint32_t has_double;           // any copy site with a doubled partner
  uint32_t pad3_;
  uint64_t lane_mask;            // the 5 pivot run bits of the lanes
  uint64_t lane_vec[5];          // run bits flipped by lane bit i
  uint64_t hi_step;              // warp slot stride (1 = contiguous walk;
                                 // > 1 = the autotuner's spread sample)
  uint32_t e_mode;               // 0 dense, 1 parity planes
  uint32_t e_parity;             // constant part of the e parity
  uint32_t row_words, e_words, plane_words;  // layout (words)
  uint32_t row_bytes;            // 4 * row_words
  uint32_t e_bytes;              // bytes per unit of e
  int32_t plane_bytes;           // bytes added when the e parity is odd
  uint32_t shift[kMaxClasses];
  uint32_t mvar[kMaxClasses];    // class bonds with lower site a loop site
                                 // and upper site not a copy site
  uint64_t mask[kMaxClasses];
  uint64_t jneg[kMaxClasses];
  uint64_t nm1[kCopyBits], jn1[kCopyBits];   // copy-site partner masks
  uint64_t nm2[kCopyBits], jn2[kCopyBits];   // (second copy of a double bond)
  uint32_t nm1v[kCopyBits], jn1v[kCopyBits]; // restricted to loop sites
  uint32_t nm2v[kCopyBits], jn2v[kCopyBits];
  int32_t degree[kCopyBits];                 // d_q
  int32_t koff[kCopies];         // constant byte offset of copy c:
                                 // popc(c) row_bytes + e_bytes unsat_cc(c)
                                 // (+ pair_bytes u_q(c) for paired copies)
  // paired copies (isd_plan_info.pair_mode): copy bit 6 (index 0) and, in
  // mode 2, copy bit 5 (index 1) are counted through pattern planes
  // instead of register copies
  uint32_t pair;                 // 0, 1, 2
  uint32_t pair_bytes[2];        // 4 * pair_words
  uint32_t pair_words[2];        // stride between pattern planes
  int32_t pair_deg[2];           // D: degree of the paired site
  int32_t pair_both;             // mode 2: extra e change of the double flip
  // Gray sites (NVRTC build only; the AOT kernel walks every loop subset
  // from scratch): the `gray` lowest loop sites are flipped one at a time
  // inside an iteration.  Per site: its loop bit, its bonds to non-copy
  // sites (masks as for the copy sites; v = restricted to loop bits), their
  // count, and the shift of each copy site's unsatisfied count when it
  // flips up (cdelta, csum = their sum).
  uint32_t gray;
  uint32_t g_mask;
  uint32_t g_bit[kMaxGray];
  uint64_t g_nm1[kMaxGray], g_jn1[kMaxGray], g_nm2[kMaxGray], g_jn2[kMaxGray];
  uint32_t g_nm1v[kMaxGray], g_jn1v[kMaxGray], g_nm2v[kMaxGray],
      g_jn2v[kMaxGray];
  int32_t g_deg[kMaxGray], g_csum[kMaxGray], g_odd[kMaxGray];
  int32_t g_cdelta[kMaxGray][kCopyBits];
  // banded tables (isd_plan_info.band_rows): rows of the table, and for a
  // launch its work items (device array of BandItem) and free run bits
  uint32_t band_rows;
  uint32_t band_free_bits;
  uint32_t band_n_items;
  uint32_t band_span;  // popcount classes per work item - 1 (plan)
  uint64_t band_items;
  // banded launches: a zeroed u32 counter the blocks claim items from
  // (dynamic scheduling; 0 = static round-robin)
  uint64_t band_claim;
  // calibration launches: device array of per-item SM cycles (0 = none)
  uint64_t band_clk;
  // banded launches: slot bits -> run bits (k1_body.cuh IsdSlotMap)
  uint32_t slot_mask[16];
  uint32_t slot_rot[16];
};

// Largest paired histogram (words): two CTAs of 512 threads per SM fit
// 28 K words each; up to 56 K words runs one CTA per SM (mode 2 only).
constexpr uint32_t kMaxPairWords = 28000;
constexpr uint32_t kMaxPair2Words = 56000;
// Banded mode-2 tables may use a block's whole shared memory (227 KB).
constexpr uint32_t kMaxBandWords = 57600;
// Work items of a banded launch span at most this many popcount classes
// of their free run bits (+1: the rows of one item = kBandSpan + 5 lane
// bits + l loop bits + (u - 2) copy bits + 1).
constexpr int kBandSpan = 2;
// one work item of a banded launch: slots [g0, g1) of the popcount-ordered
// free run bits, whose popcounts are >= q0; mirror != 0: the item's table
// holds its rows in descending order (row stride -A: the banks its lanes'
// words fall on are then those of the mirrored popcount class)
struct BandItem {
  unsigned long long g0, g1;
  unsigned int q0, mirror;
};

// ---- host side -----------------------------------------------------------
int validate_lattice(const isd_lattice* lat, char* err, size_t errlen);
// Fill `info` for the hoisted decomposition.  Returns 0 if the lattice can
// use the hoisted kernel, >0 if it is too small (canonical only).
// `ranked` (optional) receives every evaluated layout, best model estimate
// first; the C ABI times the head of that list on the GPU (capi.cu).
// `top`: configuration bits the walk holds fixed (a shard's start), seen by
// the layout model.
int compile_plan(const isd_lattice* lat, uint64_t n_configs_hint,
                 isd_plan_info* info,
                 std::vector<isd_plan_info>* ranked = nullptr,
                 uint64_t top = 0);
// run-bit count spanned by a lane mask (runs of a walk must be a multiple
// of 2^lane_span(mask) for that placement to tile the walk)
int lane_span(uint64_t lane_mask);
// lanes taking the 5 lowest run bits (valid for any launch)
void default_lanes(uint64_t* lane_mask, uint64_t* lane_vec);
int plan_loop_bits(const isd_lattice* lat, uint64_t n_configs_hint);
// one random move of the plan's lane pattern within `run_bits` run bits
bool mutate_lanes(const isd_lattice* lat, int run_bits, uint64_t* seed,
                  isd_plan_info* info);
void fill_canon(const isd_lattice* lat, CanonParams* p);
// work items of a banded launch over 2^F slots (plan.cpp; see there)
std::vector<BandItem> band_work_items(int F, int n_target, int span,
                                      const std::vector<double>& w,
                                      double flush_units, bool* exact);
// expected shared wavefronts per RED of a banded launch per segment of its
// slot order (the cost of an item, plan.cpp)
void band_slot_cost(const isd_lattice* lat, const isd_plan_info& info,
                    uint64_t run_begin, uint64_t lane_mask,
                    const uint64_t* lane_vec, int run_bits, int n_seg,
                    int samples, std::vector<double>* cost,
                    std::vector<double>* cost_mirror = nullptr,
                    const uint8_t* pos = nullptr);
// order of the free run bits in a banded launch's slots, and the slot map
// as bit fields (plan.cpp; k1_body.cuh IsdSlotMap)
void band_slot_order(const isd_lattice* lat, const isd_plan_info& info,
                     uint64_t run_begin, uint64_t lane_mask,
                     const uint64_t* lane_vec, int run_bits, bool reorder,
                     uint8_t* pos);
int band_slot_fields(const uint8_t* pos, int F, uint32_t* mask, uint32_t* rot);
void fill_hoist(const isd_lattice* lat, const isd_plan_info* info,
                HoistParams* p);

// ---- kernel launchers (enumerate.cu / thermo.cu / calibrate.cu) ----------
// Each returns the number of kernels launched, or a negative cudaError_t.
int launch_canonical(const CanonParams& p, unsigned long long* out,
                     int sm_count, void* stream, bool small_grid);
int launch_hoisted(const HoistParams& p, unsigned long long* out,
                   int sm_count, void* stream);
// threads per block (512 or 1024) and grid for a hoisted kernel
int hoisted_block(const void* fn, size_t smem, int sm_count, bool may_widen,
                  int* grid, bool banded = false);
// NVRTC-specialised k1 (jit.cpp): 1 launched, 0 unavailable (*why), <0 error
int launch_hoisted_jit(const HoistParams& p, unsigned long long* out,
                       int sm_count, void* stream, std::string* why);
// compile only (no GPU needed): cubin size, or 0 with *why
int jit_compile_check(const HoistParams& p, std::string* why);
// load P's kernel on the current device (compiling it if needed): 1 ready,
// 0 unavailable (*why)
int jit_ready(const HoistParams& p, std::string* why);
// compile (or fetch from the caches) several kernels' cubins concurrently
void jit_prefetch(const std::vector<HoistParams>& ps);
int launch_mirror(unsigned long long* t, uint32_t n, uint32_t b,
                  void* stream);
// the per-device tables of a multi-GPU walk, as seen from the root device
// (peer pointers, or local copies where peer access is unavailable)
constexpr int kMaxTables = 32;
struct TableSet {
  const unsigned long long* t[kMaxTables];
  int n;
};
int launch_gather(const TableSet& tabs, unsigned long long* sum,
                  uint32_t n_spins, uint32_t n_bonds, void* stream);
// K2 over the sum of a table set (K2a also writes that sum when `sum` is
// set; with an empty grid only the sum is formed, by K4)
int launch_thermo_set(const TableSet& tabs, unsigned long long* sum,
                      uint32_t n_spins, uint32_t n_bonds, double scale,
                      const double* fields, int n_fields, const double* temps,
                      int n_temps, double* out, void* stream);
int launch_thermo(const unsigned long long* counts, uint32_t n_spins,
                  uint32_t n_bonds, double scale, const double* fields,
                  int n_fields, const double* temps, int n_temps, double* out,
                  void* stream);
// K5, the naive cross-check engine (naive.cu): per-slot bit positions and
// an explicit bond list (slot pairs, signs); launches or -cudaError_t
int naive_enumerate(uint32_t n_spins, const uint32_t* bit_of_slot,
                    uint32_t n_bonds, const uint32_t* bond_slots,
                    const int32_t* bond_sign, int coupling_sign,
                    uint64_t start, uint64_t end, unsigned long long* out,
                    int sm_count, void* stream, std::string* why);
int run_calibration(int which, int sm_count, double* lanes_per_clk_sm,
                    double* sm_mhz);

uint64_t bump_launches(uint64_t n);

// ---- tuning knobs (knobs.cpp): set only through isd_set_knob() ----------
bool knob_known(const char* name);
bool knob_str(const char* name, std::string* out);
long knob_long(const char* name, long dflt);
std::string knob_signature();  // every knob that is set, for cache keys
int set_knob(const char* name, const char* value);
void clear_knobs();

// ---- on-disk cache (cache.cpp) -------------------------------------------
const char* build_id();
void set_cache_dirs(const std::string& colon_list);  // first one is written
std::string cache_dirs();
bool cache_get(const std::string& kind, const std::string& key,
               std::string* blob);
void cache_put(const std::string& kind, const std::string& key,
               const std::string& blob);
uint32_t hist_words_for(uint32_t nbins);
int hist_count_for(uint32_t hist_words);

}  // namespace isd
