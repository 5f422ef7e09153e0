// K2 — Z(h, T) and thermodynamics from the exact table g(M, E), fp64.
//
// Follows /root/reference/pkg/src/isingdos/thermo.py:37-88:
//   cells   = occupied (g > 0) entries, M = 2 m_idx - N, E = (2 e_idx - B)|J|
//   H       = E - h M,   x = -H / T,   shift = max over occupied cells of x
//   w       = g exp(x - shift),  s = sum w,  log Z = shift + log s,  p = w / s
//   U = p.H,  <M> = p.M,  C = p.(H-U)^2 / T^2,  chi = p.(M-<M>)^2 / T
// plus the extension <|M|> = p.|M| (BASELINE configs 2 and 5).  The
// moments are accumulated as w-weighted sums and divided by s once
// (sum(w x)/s instead of sum((w/s) x)): same value to ~1e-16 relative.
//
// One kernel; a CTA of 256 threads evaluates 4 (h, T) points, one per pair
// of warps.  The CTA first compacts the occupied bins of the table (32 KB,
// L2-resident) into shared memory — warp w takes rows m = w, w + 8, ...,
// lane j the columns e = j + 32 c, all loaded at once; one block scan of
// the per-thread counts places the cells — and keeps each row's lowest
// occupied column, so a point's H_min (the reference's shift, the max of
// x = -H/T) is a minimum over rows instead of a pass over cells.  Each pair
// of warps then evaluates its point from the cell list with warp shuffles
// and a pair barrier (no further block barrier: the kernel is latency-
// bound, and a point's critical path is what it costs).  The Boltzmann
// weight factorises over the table's axes:
//     exp(x - shift) = exp(-(E - H_min) / T) * exp(h M / T) = a_e * b_m,
// so a point needs one exponential per column and per row instead of one
// per occupied cell, and a cell costs a few DFMAs in each of the two passes
// (first moments, then central second moments).  The factors stay inside
// fp64 range while |h| N / T <= 300 (a_e, b_m <= e^300); beyond that a
// point takes one exp of the whole argument per cell.  The product differs
// from exp(x - shift) by a few ulp (the GPU tests hold every field to 1e-12
// of the reference).  The cell order is fixed and a pair's sums meet in a
// fixed order (xor-shuffle tree per warp, then warp 0 + warp 1), so a
// point's value does not depend on which other points share the launch
// (thermo_sweep(...)[0] == partition_point(...) exactly, test_thermo.py:
// 85-87).
//
// (History, c5's 702-point grid: one CTA per point over the whole table
// 42 us -> warp per point over a per-CTA compacted cell list 33 us -> one-
// CTA compaction kernel + four-warp teams 16.5 us -> one warp per point
// from a per-CTA cell list, factorised weights ~10 us -> this kernel.)
#include <cuda_runtime.h>
#include <math.h>

#include <mutex>
#include <type_traits>

#include "isd_internal.h"

namespace isd {

constexpr int kThermoThreads = 256;  // one (h, T) point per CTA
constexpr int kThermoWarps = kThermoThreads / 32;
constexpr int kColSlots = 4;         // columns per lane: B + 1 <= 128
static_assert(3 * ISD_MAX_SPINS + 1 <= 32 * kColSlots, "columns per lane");
// weights factorise while every factor stays below e^kSplitMax
constexpr double kSplitMax = 300.0;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Weight of one cell outside the factorised range (|h| N / T > 300): one
// exp of the whole argument (rare; out of line to keep the kernel small).
__device__ __noinline__ double whole_weight(double g, double en, double hmin,
                                            double t) {
  return g * exp(-(en - hmin) / t);
}

// Warps per point: a pair, so each lane walks half as many cells.
constexpr int kPairWarps = 2;
constexpr int kPointsPerCta = kThermoWarps / kPairWarps;

// Barrier over the two warps of one point (named barrier 1 + pair).
__device__ __forceinline__ void pair_sync(int pair) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(32 * kPairWarps)
               : "memory");
}

__global__ void __launch_bounds__(kThermoThreads)
    k2_thermo(const unsigned long long* __restrict__ table, uint32_t n,
              uint32_t b, double scale, const double* __restrict__ fields,
              const double* __restrict__ temps, int n_temps, int n_points,
              double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char cell_mem[];
  __shared__ int warp_tot[kThermoWarps];
  __shared__ int row_emin[ISD_MAX_SPINS + 1];  // lowest occupied e per row
  __shared__ double a_s[kPointsPerCta][32 * kColSlots];
  __shared__ double b_s[kPointsPerCta][ISD_MAX_SPINS + 1];
  __shared__ double part[kPointsPerCta][kPairWarps][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = (int)n + 1, cols = (int)b + 1;
  double* cg = reinterpret_cast<double*>(cell_mem);               // counts
  uint32_t* cme = reinterpret_cast<uint32_t*>(cg + rows * cols);  // m<<16|e

  // 1. the CTA compacts the occupied bins into shared memory: thread
  // (warp, lane) takes rows warp + 8 k and columns lane + 32 c, all loaded
  // before any is used (one L2 round trip); one block scan of the counts
  // places the cells in (warp, row slot, column slot) order.  Each row's
  // lowest occupied column is kept: H_min of a point is then a minimum
  // over rows, not over cells.
  constexpr int kRowSlots =
      (ISD_MAX_SPINS + 1 + kThermoWarps - 1) / kThermoWarps;
  unsigned long long gv[kRowSlots][kColSlots];
#pragma unroll
  for (int k = 0; k < kRowSlots; ++k) {
    const int r = warp + kThermoWarps * k;
#pragma unroll
    for (int c = 0; c < kColSlots; ++c) {
      const int e = lane + 32 * c;
      gv[k][c] = (r < rows && e < cols) ? __ldg(table + r * cols + e) : 0ull;
    }
  }
  int mine = 0;
#pragma unroll
  for (int k = 0; k < kRowSlots; ++k) {
    int emin = 0x7fffffff;
#pragma unroll
    for (int c = kColSlots - 1; c >= 0; --c) {
      mine += gv[k][c] != 0ull;
      const unsigned bal = __ballot_sync(0xffffffffu, gv[k][c] != 0ull);
      if (bal) emin = 32 * c + __ffs(bal) - 1;
    }
    const int r = warp + kThermoWarps * k;
    if (lane == 0 && r < rows) row_emin[r] = emin;
  }
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  int pos = incl - mine, nc = 0;
  for (int w = 0; w < kThermoWarps; ++w) {
    if (w < warp) pos += warp_tot[w];
    nc += warp_tot[w];
  }
#pragma unroll
  for (int k = 0; k < kRowSlots; ++k) {
#pragma unroll
    for (int c = 0; c < kColSlots; ++c) {
      if (gv[k][c] != 0ull) {
        cg[pos] = (double)gv[k][c];
        cme[pos] = ((uint32_t)(warp + kThermoWarps * k) << 16) |
                   (uint32_t)(lane + 32 * c);
        ++pos;
      }
    }
  }
  __syncthreads();

  // 2. each pair of warps evaluates one point from the shared cell list
  // (warp shuffles and a pair barrier; no further block barrier)
  const int pair = warp / kPairWarps, half = warp % kPairWarps;
  const int pl = half * 32 + lane;  // lane within the pair
  const int point = (int)blockIdx.x * kPointsPerCta + pair;
  if (point >= n_points) return;  // (both warps of the pair)
  const double h = fields[point / n_temps];
  const double t = temps[point % n_temps];
  auto cell = [&](int i, double* e, double* m, int* ei, int* mi) {
    const uint32_t me = cme[i];
    *mi = (int)(me >> 16);
    *ei = (int)(me & 0xffffu);
    *m = (double)(2 * *mi - (int)n);
    *e = (double)(2 * *ei - (int)b) * scale;
  };
  // H_min = min over rows of (lowest occupied E) - h M; shift = -H_min / T
  // (= max of x = -H / T: division by T > 0 is monotone).  Both warps of
  // the pair compute it, identically.
  double hmin = INFINITY;
  for (int r = lane; r < rows; r += 32)
    if (row_emin[r] != 0x7fffffff)
      hmin = fmin(hmin, (double)(2 * row_emin[r] - (int)b) * scale -
                            h * (double)(2 * r - (int)n));
  hmin = warp_min(hmin);
  const double shift = -hmin / t;
  const bool split = fabs(h) * (double)n / t <= kSplitMax;
  if (split) {
    for (int j = pl; j < cols; j += 32 * kPairWarps)
      a_s[pair][j] = exp(-((double)(2 * j - (int)b) * scale - hmin) / t);
    if (pl < rows) b_s[pair][pl] = exp(h * (double)(2 * pl - (int)n) / t);
    pair_sync(pair);
  }
  // the pair's sums: each warp's xor-tree total, then warp 0 + warp 1
  auto pair_sum = [&](auto nv_const, double* v) {
    constexpr int NV = decltype(nv_const)::value;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) part[pair][half][k] = v[k];
    }
    pair_sync(pair);
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = part[pair][0][k] + part[pair][1][k];
    pair_sync(pair);  // (part is reused by the next sum)
  };
  // pass 1: s = sum w and the first moments as w-weighted sums
  double red[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i = pl; i < nc; i += 32 * kPairWarps) {
    double e, m;
    int ei, mi;
    cell(i, &e, &m, &ei, &mi);
    const double en = e - h * m;
    const double w = split ? cg[i] * a_s[pair][ei] * b_s[pair][mi]
                           : whole_weight(cg[i], en, hmin, t);
    red[0] += w;
    red[1] += w * en;
    red[2] += w * m;
    red[3] += w * fabs(m);
  }
  pair_sum(std::integral_constant<int, 4>{}, red);
  const double s = red[0];
  const double u = red[1] / s;
  const double mean_m = red[2] / s;
  const double mean_abs = red[3] / s;
  // pass 2: central second moments (the two-pass form of thermo.py:75-77;
  // the raw <H^2> - <H>^2 form cancels catastrophically at low T)
  red[0] = red[1] = 0.0;
  for (int i = pl; i < nc; i += 32 * kPairWarps) {
    double e, m;
    int ei, mi;
    cell(i, &e, &m, &ei, &mi);
    const double en = e - h * m;
    const double w = split ? cg[i] * a_s[pair][ei] * b_s[pair][mi]
                           : whole_weight(cg[i], en, hmin, t);
    const double de = en - u, dm = m - mean_m;
    red[0] += w * (de * de);
    red[1] += w * (dm * dm);
  }
  pair_sum(std::integral_constant<int, 2>{}, red);
  const double ve = red[0] / s;
  const double vm = red[1] / s;
  if (pl == 0) {
    const double log_z = shift + log(s);
    double* o = out + (size_t)point * ISD_THERMO_FIELDS;
    o[0] = log_z;
    o[1] = -t * log_z;
    o[2] = u;
    o[3] = ve / (t * t);
    o[4] = mean_m;
    o[5] = vm / t;
    o[6] = mean_abs;
  }
}

// K4: the combined table of several devices' tables (peer reads over
// NVLink), for a multi-GPU walk that is not followed by K2.
__global__ void __launch_bounds__(256)
    k4_gather(const TableSet tabs, unsigned long long* __restrict__ sum,
              uint32_t nbins) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbins) return;
  unsigned long long g = 0;
  for (int t = 0; t < tabs.n; ++t) g += tabs.t[t][i];
  sum[i] = g;
}

int launch_gather(const TableSet& tabs, unsigned long long* sum,
                  uint32_t n_spins, uint32_t n_bonds, void* stream) {
  const uint32_t nbins = (n_spins + 1) * (n_bonds + 1);
  k4_gather<<<(nbins + 255) / 256, 256, 0, (cudaStream_t)stream>>>(tabs, sum,
                                                                   nbins);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 1 : -(int)e;
}

int launch_thermo(const unsigned long long* counts, uint32_t n_spins,
                  uint32_t n_bonds, double scale, const double* fields,
                  int n_fields, const double* temps, int n_temps, double* out,
                  void* stream) {
  TableSet one;
  one.n = 1;
  one.t[0] = counts;
  return launch_thermo_set(one, nullptr, n_spins, n_bonds, scale, fields,
                           n_fields, temps, n_temps, out, stream);
}

// K2 over the sum of a table set: one table is read in place; several are
// first summed by K4 (each read once, e.g. over NVLink) into `sum`, or into
// stream-ordered scratch when the caller wants no sum.
int launch_thermo_set(const TableSet& tabs, unsigned long long* sum,
                      uint32_t n_spins, uint32_t n_bonds, double scale,
                      const double* fields, int n_fields, const double* temps,
                      int n_temps, double* out, void* stream) {
  const int points = n_fields * n_temps;
  cudaStream_t st = (cudaStream_t)stream;
  int launched = 0;
  const unsigned long long* table = tabs.t[0];
  void* scratch = nullptr;
  if (tabs.n > 1 || sum) {
    unsigned long long* dst = sum;
    if (!dst) {
      // stream-ordered scratch, kept in the device's default pool
      // (threshold 64 MiB) so steady calls do not go back to the driver
      static std::once_flag pool_ready[64];
      int dev = 0;
      cudaGetDevice(&dev);
      if (dev < 64)
        std::call_once(pool_ready[dev], [dev] {
          cudaMemPool_t pool;
          if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = 64ull << 20;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold,
                                    &thr);
          }
          cudaGetLastError();
        });
      const size_t bytes = (size_t)(n_spins + 1) * (n_bonds + 1) * 8;
      cudaError_t e = cudaMallocAsync(&scratch, bytes, st);
      if (e != cudaSuccess) return -(int)e;
      dst = reinterpret_cast<unsigned long long*>(scratch);
    }
    const int r = launch_gather(tabs, dst, n_spins, n_bonds, st);
    if (r < 0) return r;
    launched += r;
    table = dst;
  }
  if (points > 0) {
    // the CTA's cell list: 12 bytes per bin of the table
    const size_t smem = (size_t)(n_spins + 1) * (n_bonds + 1) * 12;
    static std::once_flag attr_set[64];  // (a per-device attribute)
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(attr_set[dev & 63], [] {
      cudaFuncSetAttribute(
          k2_thermo, cudaFuncAttributeMaxDynamicSharedMemorySize,
          (int)((ISD_MAX_SPINS + 1) * (3 * ISD_MAX_SPINS + 1) * 12));
    });
    const int grid = (points + kPointsPerCta - 1) / kPointsPerCta;
    k2_thermo<<<grid, kThermoThreads, smem, st>>>(table, n_spins, n_bonds,
                                                  scale, fields, temps,
                                                  n_temps, points, out);
    ++launched;
  }
  cudaError_t e = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? launched : -(int)e;
}

}  // namespace isd
