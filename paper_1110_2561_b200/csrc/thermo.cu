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
// K2a compacts the occupied cells of the table once, in table order (a
// block prefix scan); K2b gives each (h, T) point one CTA that walks the
// cell list; each lane takes a fixed strided subset and the partials meet
// in a fixed xor-shuffle tree.  A point's result therefore does not depend on which other points
// share the launch (thermo_sweep(...)[0] == partition_point(...) exactly,
// test_thermo.py:85-87).
#include <cuda_runtime.h>
#include <math.h>

#include <mutex>

#include "isd_internal.h"

namespace isd {

constexpr int kThermoThreads = 256;  // one (h, T) point per CTA, 8 warps
constexpr int kKeep = 8;  // cells per lane kept in registers (2048 cells)
constexpr int kMaxBins = (ISD_MAX_SPINS + 1) * (3 * ISD_MAX_SPINS + 1);

struct Cell {
  double g;  // count (exact in fp64 below 2^53)
  float m;   // M = 2 m_idx - N
  int e;     // 2 e_idx - B (E = e * |J|)
};

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

// K2a: compact the occupied cells of the table, in table order, into a
// scratch list (one CTA, <= 5 bins per thread, shuffle scans).
constexpr int kCompactThreads = 1024;
static_assert(kMaxBins <= 5 * kCompactThreads, "<= 5 bins per thread");

// K2a sums its input over up to kMaxTables tables (the per-device tables of
// a multi-GPU walk, read over NVLink peer access) and, when `sum` is set,
// writes the combined table there: the cross-device reduce is fused into the
// compaction the thermodynamics needs anyway.
__global__ void __launch_bounds__(kCompactThreads)
    k2_compact(const TableSet tabs, unsigned long long* __restrict__ sum,
               uint32_t n, uint32_t b, Cell* __restrict__ cells,
               int* __restrict__ n_cells) {
  __shared__ int warp_tot[kCompactThreads / 32];
  const uint32_t stride = b + 1;
  const uint32_t nbins = (n + 1) * stride;
  const uint32_t per = (nbins + kCompactThreads - 1) / kCompactThreads;  // <= 5
  const uint32_t lo = threadIdx.x * per;
  unsigned long long g[5];
  int mine = 0;
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const uint32_t i = lo + j;
    g[j] = 0ull;
    if (j < (int)per && i < nbins) {
      for (int t = 0; t < tabs.n; ++t) g[j] += tabs.t[t][i];
      if (sum) sum[i] = g[j];
    }
    mine += g[j] != 0;
  }
  // exclusive prefix of `mine` over the CTA: warp shuffle scan, then the
  // warp totals scanned by warp 0
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += v;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  int pos = (warp ? warp_tot[warp - 1] : 0) + incl - mine;
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    if (!g[j]) continue;
    const uint32_t i = lo + j;
    const int mi = (int)(i / stride), ei = (int)(i - mi * stride);
    cells[pos].g = (double)g[j];
    cells[pos].m = (float)(2 * mi - (int)n);
    cells[pos].e = 2 * ei - (int)b;
    ++pos;
  }
  if (threadIdx.x == kCompactThreads - 1) *n_cells = warp_tot[31];
}

// K2b: the observables, one CTA of 256 threads per (h, T) point.  Each lane
// holds its (up to kKeep) cells' energy, count and weight in registers
// across the three passes, and every pass ends in one block reduction (a
// fixed xor-shuffle tree per warp, then the 8 warp partials in a fixed
// order), so a point's value does not depend on the grid it is in.
// (History: a four-warp team per point re-read its ~9 cells per lane from
// L2 in every pass; the whole-CTA point keeps them: 11.4 -> ~4 us on c5.)
__global__ void __launch_bounds__(kThermoThreads)
    k2_thermo(const Cell* __restrict__ cells, const int* __restrict__ n_cells,
              double scale, const double* __restrict__ fields,
              const double* __restrict__ temps, int n_temps, int n_points,
              double* __restrict__ out) {
  constexpr int kWarps = kThermoThreads / 32;
  __shared__ double part[kWarps][4];
  const int nc = *n_cells;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tl = threadIdx.x;
  const int point = blockIdx.x;
  if (point >= n_points) return;  // (uniform per CTA)
  const double h = fields[point / n_temps];
  const double t = temps[point % n_temps];
  // block reduction of NV values (sum, or min when `is_min`)
  auto block_reduce = [&](double* v, int nv, bool is_min) {
    for (int k = 0; k < nv; ++k)
      v[k] = is_min ? warp_min(v[k]) : warp_sum(v[k]);
    if (lane == 0)
      for (int k = 0; k < nv; ++k) part[warp][k] = v[k];
    __syncthreads();
    for (int k = 0; k < nv; ++k) {
      double r = part[0][k];
#pragma unroll
      for (int w = 1; w < kWarps; ++w)
        r = is_min ? fmin(r, part[w][k]) : r + part[w][k];
      v[k] = r;
    }
    __syncthreads();
  };

  // pass 1: each lane's cells (energy H = E - h M kept), shift = max of
  // x = -H / T = -H_min / T (division by T > 0 is monotone: one division)
  double en[kKeep], mm[kKeep], gg[kKeep];
  double red[4];
  red[0] = INFINITY;
#pragma unroll
  for (int j = 0; j < kKeep; ++j) {
    const int i = tl + kThermoThreads * j;
    en[j] = 0.0;
    mm[j] = 0.0;
    gg[j] = 0.0;
    if (i < nc) {
      const Cell c = cells[i];
      mm[j] = (double)c.m;
      en[j] = (double)c.e * scale - h * mm[j];
      gg[j] = c.g;
      red[0] = fmin(red[0], en[j]);
    }
  }
  for (int i = tl + kThermoThreads * kKeep; i < nc; i += kThermoThreads) {
    const double m = (double)cells[i].m;
    red[0] = fmin(red[0], (double)cells[i].e * scale - h * m);
  }
  block_reduce(red, 1, true);
  const double shift = -red[0] / t;

  // pass 2: w = g exp(x - shift); s = sum w and the first moments as
  // w-weighted sums (divided by s afterwards)
  double wk[kKeep];
  red[0] = red[1] = red[2] = red[3] = 0.0;
#pragma unroll
  for (int j = 0; j < kKeep; ++j) {
    // (off the list: no exp — exp(-shift) alone may overflow)
    wk[j] = gg[j] != 0.0 ? gg[j] * exp(-en[j] / t - shift) : 0.0;
    red[0] += wk[j];
    red[1] += wk[j] * en[j];
    red[2] += wk[j] * mm[j];
    red[3] += wk[j] * fabs(mm[j]);
  }
  for (int i = tl + kThermoThreads * kKeep; i < nc; i += kThermoThreads) {
    const double m = (double)cells[i].m;
    const double e = (double)cells[i].e * scale - h * m;
    const double w = cells[i].g * exp(-e / t - shift);
    red[0] += w;
    red[1] += w * e;
    red[2] += w * m;
    red[3] += w * fabs(m);
  }
  block_reduce(red, 4, false);
  const double s = red[0];
  const double u = red[1] / s;
  const double mean_m = red[2] / s;
  const double mean_abs = red[3] / s;

  // pass 3: central second moments (the two-pass form of thermo.py:75-77;
  // the raw <H^2> - <H>^2 form cancels catastrophically at low T)
  red[0] = red[1] = 0.0;
#pragma unroll
  for (int j = 0; j < kKeep; ++j) {
    const double de = en[j] - u, dm = mm[j] - mean_m;
    red[0] += wk[j] * (de * de);
    red[1] += wk[j] * (dm * dm);
  }
  for (int i = tl + kThermoThreads * kKeep; i < nc; i += kThermoThreads) {
    const double m = (double)cells[i].m;
    const double e = (double)cells[i].e * scale - h * m;
    const double w = cells[i].g * exp(-e / t - shift);
    const double de = e - u, dm = m - mean_m;
    red[0] += w * (de * de);
    red[1] += w * (dm * dm);
  }
  block_reduce(red, 2, false);
  const double ve = red[0] / s;
  const double vm = red[1] / s;

  if (tl == 0) {
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

int launch_thermo_set(const TableSet& tabs, unsigned long long* sum,
                      uint32_t n_spins, uint32_t n_bonds, double scale,
                      const double* fields, int n_fields, const double* temps,
                      int n_temps, double* out, void* stream) {
  const int points = n_fields * n_temps;
  if (points <= 0) {
    if (sum) return launch_gather(tabs, sum, n_spins, n_bonds, stream);
    return 0;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bins = (size_t)(n_spins + 1) * (n_bonds + 1);
  // stream-ordered scratch: safe for concurrent calls on different streams.
  // Keep freed blocks in the device's default pool (threshold 64 MiB) so a
  // steady stream of calls does not go back to the driver every time.
  static std::once_flag pool_ready[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64)
    std::call_once(pool_ready[dev], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = 64ull << 20;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
    });
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(Cell) * bins + 16, st);
  if (e != cudaSuccess) return -(int)e;
  Cell* cells = reinterpret_cast<Cell*>(scratch);
  int* n_cells = reinterpret_cast<int*>(reinterpret_cast<char*>(scratch) +
                                        sizeof(Cell) * bins);
  k2_compact<<<1, kCompactThreads, 0, st>>>(tabs, sum, n_spins, n_bonds,
                                            cells, n_cells);
  const int grid = points;
  k2_thermo<<<grid, kThermoThreads, 0, st>>>(cells, n_cells, scale, fields,
                                             temps, n_temps, points, out);
  e = cudaGetLastError();
  cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? 2 : -(int)e;
}

}  // namespace isd
