// K1 — exhaustive enumeration of Ising configurations into g(M, E) on sm_100a.
//
// Replaces the reference's batch loop
//   enumerate_shard -> _classify_batch -> np.bincount
//   (/root/reference/pkg/src/isingdos/enumeration.py:167-235)
// with two integer kernels that share one histogram scheme:
//
//  * k1_canonical: one thread per configuration index (grid-stride), the
//    full bond-class evaluation per index:
//        m = popc(x),  e = sum_c popc(((x ^ x>>s_c) ^ jneg_c) & bond_c)
//    Used for ranges not aligned to a run and for tiny lattices, and kept
//    as the measured "canonical formulation" baseline.
//
//  * k1_hoisted: every configuration is still counted individually, but the
//    work that does not change between neighbouring indices is hoisted:
//    bits [k, N) are fixed per thread ("run"), the loop sites of [0, k) are
//    the thread's loop, and 7 copy sites of [0, k) are 128 register copies.
//    Per group of 128 copies the kernel evaluates the loop-dependent bonds
//    with LOP3/POPC over precomputed masks and derives each copy site's
//    flip cost delta_q = d_q - 2 n_q; each copy's histogram address is then
//    one add (subset sum over the copy bits) plus a per-lattice constant
//    offset folded into the shared-memory reduction.  The body lives in
//    k1_body.cuh and is also compiled per lattice with NVRTC (jit.cpp).
//
// Counts go to shared-memory u32 histograms (one per group of warps),
// flushed once per block into the per-GPU uint64 table with 64-bit global
// atomics.  The host bounds the configurations per launch so no u32 counter
// can wrap (capi.cu).
#include <cuda_runtime.h>

#include "isd_internal.h"

// Debug builds (-DISD_DEBUG_BOUNDS, libisingdos_b200_dbg.so) trap on any
// histogram address outside the warp's own histogram: the bounds check that
// stands in for compute-sanitizer, which is closed on the GPU pool.
#ifdef ISD_DEBUG_BOUNDS
#define ISD_CHECK_ADDR(a, lo, bytes)                                  \
  do {                                                                \
    if ((uint32_t)((a) - (lo)) >= (bytes) || ((a) & 3u)) __trap();    \
  } while (0)
#else
#define ISD_CHECK_ADDR(a, lo, bytes) \
  do {                               \
  } while (0)
#endif

#include "k1_body.cuh"

#ifndef ISD_HOIST_PART
#define ISD_HOIST_PART 0
#endif

namespace isd {
#if ISD_HOIST_PART == 0


__device__ __forceinline__ void red_shared_inc(uint32_t addr) {
  isd_red_shared_inc(addr);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Zero the block's histograms.
__device__ __forceinline__ void zero_hist(uint32_t* hist, uint32_t words) {
  uint4* h4 = reinterpret_cast<uint4*>(hist);
  const uint32_t n4 = words / 4;
  for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x)
    h4[i] = make_uint4(0, 0, 0, 0);
}

// Sum the block's histograms and add the nonzero bins to the global table.
__device__ __forceinline__ void flush_hist(const uint32_t* hist,
                                           uint32_t n_hist,
                                           uint32_t hist_words, uint32_t nbins,
                                           unsigned long long* out) {
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) {
    unsigned long long s = 0;
    for (uint32_t h = 0; h < n_hist; ++h) s += hist[h * hist_words + b];
    if (s) atomicAdd(out + b, s);
  }
}

// ---------------------------------------------------------------------------
// canonical kernel
// ---------------------------------------------------------------------------
template <int NC, bool WIDE>
__global__ void __launch_bounds__(kThreads)
    k1_canonical(const __grid_constant__ CanonParams P,
                 unsigned long long* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t hist[];
  zero_hist(hist, P.n_hist * P.hist_words);
  __syncthreads();
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t hbase =
      smem_addr(hist + (warp % P.n_hist) * P.hist_words);
  const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = P.start + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
       x < P.end; x += gstride) {
    uint32_t m, e = 0;
    if constexpr (WIDE) {
      m = __popcll(x);
#pragma unroll
      for (int c = 0; c < NC; ++c)
        e += __popcll(((x ^ (x >> P.shift[c])) ^ P.jneg[c]) & P.mask[c]);
    } else {
      const uint32_t y = (uint32_t)x;
      m = __popc(y);
#pragma unroll
      for (int c = 0; c < NC; ++c)
        e += __popc(((y ^ (y >> P.shift[c])) ^ (uint32_t)P.jneg[c]) &
                    (uint32_t)P.mask[c]);
    }
    ISD_CHECK_ADDR(hbase + 4u * (m * P.stride + e), hbase, 4u * P.nbins);
    red_shared_inc(hbase + 4u * (m * P.stride + e));
  }
  __syncthreads();
  flush_hist(hist, P.n_hist, P.hist_words, P.nbins, out);
}

#endif  // ISD_HOIST_PART == 0

// ---------------------------------------------------------------------------
// hoisted kernel (ahead-of-time build; body in k1_body.cuh)
// ---------------------------------------------------------------------------
struct RuntimeTraits {
  const HoistParams& P;
  __device__ uint32_t k() const { return P.k; }
  __device__ uint32_t nloop() const { return 1u << P.l; }
  __device__ uint64_t above_k() const { return P.above_k; }
  __device__ uint64_t odd_mask() const { return P.odd_mask; }
  __device__ uint32_t loop_mask() const { return P.loop_mask; }
  __device__ uint32_t e_parity() const { return P.e_parity; }
  __device__ uint32_t e_mode() const { return P.e_mode; }
  __device__ uint32_t row_bytes() const { return P.row_bytes; }
  __device__ uint32_t e_bytes() const { return P.e_bytes; }
  __device__ int32_t plane_bytes() const { return P.plane_bytes; }
  __device__ uint32_t row_words() const { return P.row_words; }
  __device__ uint32_t e_words() const { return P.e_words; }
  __device__ uint32_t plane_words() const { return P.plane_words; }
  __device__ uint32_t stride() const { return P.stride; }
  __device__ uint32_t nbins() const { return P.nbins; }
  __device__ uint32_t hist_words() const { return P.hist_words; }
  __device__ uint32_t n_hist() const { return P.n_hist; }
  __device__ uint32_t shift(int c) const { return P.shift[c]; }
  __device__ uint64_t mask(int c) const { return P.mask[c]; }
  __device__ uint64_t jneg(int c) const { return P.jneg[c]; }
  __device__ uint32_t mvar(int c) const { return P.mvar[c]; }
  __device__ uint64_t nm1(int q) const { return P.nm1[q]; }
  __device__ uint64_t jn1(int q) const { return P.jn1[q]; }
  __device__ uint64_t nm2(int q) const { return P.nm2[q]; }
  __device__ uint64_t jn2(int q) const { return P.jn2[q]; }
  __device__ uint32_t nm1v(int q) const { return P.nm1v[q]; }
  __device__ uint32_t jn1v(int q) const { return P.jn1v[q]; }
  __device__ uint32_t nm2v(int q) const { return P.nm2v[q]; }
  __device__ uint32_t jn2v(int q) const { return P.jn2v[q]; }
  __device__ int32_t degree(int q) const { return P.degree[q]; }
  __device__ uint32_t koff(int c) const { return (uint32_t)P.koff[c]; }
  __device__ uint32_t pair_bytes(int i) const { return P.pair_bytes[i]; }
  __device__ uint32_t pair_words(int i) const { return P.pair_words[i]; }
  __device__ int32_t pair_deg(int i) const { return P.pair_deg[i]; }
  __device__ int32_t pair_both() const { return P.pair_both; }
  // no Gray sites in the ahead-of-time build (the stubs are never called)
  __device__ uint32_t band_rows() const { return P.band_rows; }
  __host__ __device__ static constexpr int gray() { return 0; }
  // (mode 3's external degree is a run-time value here: direct flush)
  __host__ __device__ static constexpr int tri_r() { return -1; }
  __device__ uint32_t g_mask() const { return 0; }
  __device__ uint32_t g_bit(int) const { return 0; }
  __device__ uint64_t g_nm1(int) const { return 0; }
  __device__ uint64_t g_jn1(int) const { return 0; }
  __device__ uint64_t g_nm2(int) const { return 0; }
  __device__ uint64_t g_jn2(int) const { return 0; }
  __device__ uint32_t g_nm1v(int) const { return 0; }
  __device__ uint32_t g_jn1v(int) const { return 0; }
  __device__ uint32_t g_nm2v(int) const { return 0; }
  __device__ uint32_t g_jn2v(int) const { return 0; }
  __device__ int32_t g_deg(int) const { return 0; }
  __device__ int32_t g_csum(int) const { return 0; }
  __device__ int32_t g_odd(int) const { return 0; }
  __device__ int32_t g_cdelta(int, int) const { return 0; }
};

// (mode-2 histograms can be too large for two blocks per SM: those kernels
// may run 1024-thread blocks, which caps them at 64 registers)
template <int NC, bool DOUBLE, int PAIR>
__global__ void __launch_bounds__(PAIR >= 2 ? kWideThreads : kThreads)
    k1_hoisted(const __grid_constant__ HoistParams P,
               unsigned long long* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t hist[];
  const RuntimeTraits L{P};
  IsdLanes lanes;
#pragma unroll
  for (int i = 0; i < 5; ++i) lanes.v[i] = P.lane_vec[i];
  IsdSlotMap smap;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    smap.mask[j] = P.slot_mask[j];
    smap.rot[j] = P.slot_rot[j];
  }
  k1_hoisted_body<NC, DOUBLE, PAIR>(
      L, P.run_begin, P.run_end - P.run_begin, P.hi_step, P.lane_mask, lanes,
      reinterpret_cast<const IsdBandItem*>(P.band_items), P.band_n_items,
      (int)P.band_free_bits,
      reinterpret_cast<unsigned int*>(P.band_claim), smap,
      reinterpret_cast<unsigned long long*>(P.band_clk), hist, out);
}

#if ISD_HOIST_PART == 0
// ---------------------------------------------------------------------------
// flip-symmetry completion: rows m and N-m both become their sum
// ---------------------------------------------------------------------------
__global__ void k3_mirror(unsigned long long* __restrict__ t, uint32_t n,
                          uint32_t stride) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t half_rows = n / 2 + 1;  // rows 0..n/2
  if (i >= half_rows * stride) return;
  const uint32_t m = i / stride, e = i - m * stride;
  const uint32_t mm = n - m;
  if (mm < m) return;
  const unsigned long long a = t[m * stride + e];
  if (mm == m) {
    t[m * stride + e] = 2 * a;
  } else {
    const unsigned long long b = t[mm * stride + e];
    t[m * stride + e] = a + b;
    t[mm * stride + e] = a + b;
  }
}

int launch_mirror(unsigned long long* t, uint32_t n, uint32_t b,
                  void* stream) {
  const uint32_t stride = b + 1;
  const uint32_t work = (n / 2 + 1) * stride;
  k3_mirror<<<(work + 255) / 256, 256, 0, (cudaStream_t)stream>>>(t, n, stride);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 1 : -(int)e;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int blocks_for(const void* fn, size_t smem, int sm_count) {
  int per_sm = 0;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads,
                                                    smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return per_sm * sm_count;
}

template <int NC, bool W>
static int launch_canon_t(const CanonParams& p, unsigned long long* out,
                          int sm_count, cudaStream_t st, bool small_grid) {
  const size_t smem = (size_t)p.n_hist * p.hist_words * 4;
  const void* fn = (const void*)k1_canonical<NC, W>;
  int grid = blocks_for(fn, smem, sm_count);
  const uint64_t n = p.end - p.start;
  if (small_grid) {
    const uint64_t need = (n + kThreads - 1) / kThreads;
    if (need < (uint64_t)grid) grid = (int)(need ? need : 1);
  }
  k1_canonical<NC, W><<<grid, kThreads, smem, st>>>(p, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 1 : -(int)e;
}

int launch_canonical(const CanonParams& p, unsigned long long* out,
                     int sm_count, void* stream, bool small_grid) {
  cudaStream_t st = (cudaStream_t)stream;
  // The 32-bit path is exact only when every site (and every bond) lives in
  // the low word.
  const bool wide = p.n_spins > 32;
  switch (p.n_classes) {
#define CASE(NC)                                                              \
  case NC:                                                                    \
    return wide ? launch_canon_t<NC, true>(p, out, sm_count, st, small_grid)  \
                : launch_canon_t<NC, false>(p, out, sm_count, st, small_grid);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default:
      return -(int)cudaErrorInvalidValue;
  }
}

// Threads per block of the hoisted kernel: 512, or 1024 when a histogram
// this large leaves room for one block per SM (twice the warps to hide the
// issue latency).  The grid is one wave of resident blocks.
// A banded launch deals one work item to each block: one block of 1024
// threads per SM even where two of 512 would fit (c3's 95 KB table: the
// hardware placed consecutive blocks — the ones holding items — in pairs,
// leaving half the SMs idle).
int hoisted_block(const void* fn, size_t smem, int sm_count, bool may_widen,
                  int* grid, bool banded) {
  int threads = kThreads;
  int per_sm = 0;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads,
                                                    smem) != cudaSuccess)
    per_sm = 1;
  if ((per_sm <= 1 || banded) && may_widen) {
    int wide = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wide, fn, kWideThreads,
                                                      smem) == cudaSuccess &&
        wide >= 1) {
      threads = kWideThreads;
      per_sm = 1;
    }
  }
  if (per_sm < 1) per_sm = 1;
  cudaGetLastError();
  *grid = per_sm * sm_count;
  return threads;
}

#endif  // ISD_HOIST_PART == 0

template <int NC, bool D, int PR>
static int launch_hoist_t(const HoistParams& p, unsigned long long* out,
                          int sm_count, cudaStream_t st) {
  const size_t smem = (size_t)p.n_hist * p.hist_words * 4;
  const void* fn = (const void*)k1_hoisted<NC, D, PR>;
  int grid = 0;
  const int threads =
      hoisted_block(fn, smem, sm_count, PR >= 2, &grid, p.band_rows > 0);
  const uint64_t runs = p.run_end - p.run_begin;
  const uint64_t need = (runs + threads - 1) / threads;
  if (need < (uint64_t)grid) grid = (int)(need ? need : 1);
  k1_hoisted<NC, D, PR><<<grid, threads, smem, st>>>(p, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 1 : -(int)e;
}

// The hoisted kernel's instantiations (8 class counts x double bonds x 4
// pairing modes) are split over four translation units by class count —
// the build compiles this file once per ISD_HOIST_PART = 0..3 in parallel;
// part p holds NC = 2p + 1 and 2p + 2, part 0 also everything else here.
#define ISD_PART_NAME2(p) launch_hoisted_part##p
#define ISD_PART_NAME(p) ISD_PART_NAME2(p)
int ISD_PART_NAME(ISD_HOIST_PART)(const HoistParams& p,
                                  unsigned long long* out, int sm_count,
                                  cudaStream_t st) {
  const bool dbl = p.has_double != 0;
  switch (p.n_classes * 4 + (p.pair > 3 ? 0 : p.pair)) {
#define CASE1(NC, PR)                                                  \
  case (NC) * 4 + PR:                                                  \
    return dbl ? launch_hoist_t<(NC), true, PR>(p, out, sm_count, st)  \
               : launch_hoist_t<(NC), false, PR>(p, out, sm_count, st);
#define CASE(NC) CASE1(NC, 0) CASE1(NC, 1) CASE1(NC, 2) CASE1(NC, 3)
    CASE(2 * ISD_HOIST_PART + 1) CASE(2 * ISD_HOIST_PART + 2)
#undef CASE
#undef CASE1
    default:
      return -(int)cudaErrorInvalidValue;
  }
}

#if ISD_HOIST_PART == 0
int launch_hoisted_part1(const HoistParams&, unsigned long long*, int,
                         cudaStream_t);
int launch_hoisted_part2(const HoistParams&, unsigned long long*, int,
                         cudaStream_t);
int launch_hoisted_part3(const HoistParams&, unsigned long long*, int,
                         cudaStream_t);

int launch_hoisted(const HoistParams& p, unsigned long long* out, int sm_count,
                   void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch ((p.n_classes - 1) / 2) {
    case 0: return launch_hoisted_part0(p, out, sm_count, st);
    case 1: return launch_hoisted_part1(p, out, sm_count, st);
    case 2: return launch_hoisted_part2(p, out, sm_count, st);
    case 3: return launch_hoisted_part3(p, out, sm_count, st);
    default: return -(int)cudaErrorInvalidValue;
  }
}
#endif

}  // namespace isd
