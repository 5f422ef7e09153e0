// K2 — Z(h, T) and thermodynamics from the exact table g(M, E), fp64.
//
// Follows /root/reference/pkg/src/isingdos/thermo.py:37-88 step for step:
//   cells   = occupied (g > 0) entries, M = 2 m_idx - N, E = (2 e_idx - B)|J|
//   H       = E - h M,   x = -H / T,   shift = max over occupied cells of x
//   w       = g exp(x - shift),  s = sum w,  log Z = shift + log s,  p = w / s
//   U = p.H,  <M> = p.M,  C = p.(H-U)^2 / T^2,  chi = p.(M-<M>)^2 / T
// plus the extension <|M|> = p.|M| (BASELINE configs 2 and 5).
//
// One warp per (h, T) point, four points per CTA.  The CTA first compacts
// the occupied cells of the table into shared memory, in table order (warp
// ballots + a CTA prefix per chunk), so every warp walks the same cell list; each lane
// takes a fixed strided subset and the partials meet in a fixed xor-shuffle
// tree.  A point's result therefore does not depend on which other points
// share the launch (thermo_sweep(...)[0] == partition_point(...) exactly,
// test_thermo.py:85-87).
#include <cuda_runtime.h>
#include <math.h>

#include "isd_internal.h"

namespace isd {

constexpr int kThermoThreads = 128;                 // 4 warps = 4 points
constexpr int kThermoPoints = kThermoThreads / 32;
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

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(kThermoThreads)
    k2_thermo(const unsigned long long* __restrict__ counts, uint32_t n,
              uint32_t b, double scale, const double* __restrict__ fields,
              const double* __restrict__ temps, int n_temps, int n_points,
              double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  Cell* cells = reinterpret_cast<Cell*>(smem);
  const uint32_t stride = b + 1;
  const uint32_t nbins = (n + 1) * stride;

  // ---- compact the occupied cells, in table order ----
  // chunks of kThermoThreads bins: coalesced loads, warp ballots for the
  // in-warp prefix, per-warp totals for the CTA prefix
  __shared__ int warp_tot[kThermoPoints];
  const int lane_id = threadIdx.x & 31, warp_id = threadIdx.x >> 5;
  int base = 0;
  for (uint32_t c0 = 0; c0 < nbins; c0 += kThermoThreads) {
    const uint32_t i = c0 + threadIdx.x;
    const unsigned long long g = i < nbins ? counts[i] : 0ull;
    const unsigned int ball = __ballot_sync(0xffffffffu, g != 0);
    if (lane_id == 0) warp_tot[warp_id] = __popc(ball);
    __syncthreads();
    int before = base;
    for (int w = 0; w < warp_id; ++w) before += warp_tot[w];
    if (g) {
      const int pos = before + __popc(ball & ((1u << lane_id) - 1));
      const int mi = (int)(i / stride), ei = (int)(i - mi * stride);
      cells[pos].g = (double)g;
      cells[pos].m = (float)(2 * mi - (int)n);
      cells[pos].e = 2 * ei - (int)b;
    }
    for (int w = 0; w < kThermoPoints; ++w) base += warp_tot[w];
    __syncthreads();
  }
  const int nc = base;

  const int point = blockIdx.x * kThermoPoints + (threadIdx.x >> 5);
  if (point >= n_points) return;
  const int lane = threadIdx.x & 31;
  const double h = fields[point / n_temps];
  const double t = temps[point % n_temps];

  // pass 1: shift = max x over occupied cells
  double xmax = -INFINITY;
  for (int i = lane; i < nc; i += 32) {
    const double m = (double)cells[i].m;
    const double e = (double)cells[i].e * scale;
    const double en = e - h * m;
    xmax = fmax(xmax, -en / t);
  }
  const double shift = warp_max(xmax);

  // pass 2: s = sum g exp(x - shift).  Two accumulators per lane (cells
  // i and i + 32 of each 64-cell stripe) for ILP; fixed combination order.
  double s0 = 0.0, s1 = 0.0;
  for (int i = lane; i < nc; i += 64) {
    {
      const double m = (double)cells[i].m;
      const double e = (double)cells[i].e * scale;
      s0 += cells[i].g * exp(-(e - h * m) / t - shift);
    }
    if (i + 32 < nc) {
      const double m = (double)cells[i + 32].m;
      const double e = (double)cells[i + 32].e * scale;
      s1 += cells[i + 32].g * exp(-(e - h * m) / t - shift);
    }
  }
  const double s = warp_sum(s0 + s1);

  // pass 3: first moments
  double u = 0.0, mean_m = 0.0, mean_abs = 0.0;
  for (int i = lane; i < nc; i += 32) {
    const double m = (double)cells[i].m;
    const double e = (double)cells[i].e * scale;
    const double en = e - h * m;
    const double p = (cells[i].g * exp(-en / t - shift)) / s;
    u += p * en;
    mean_m += p * m;
    mean_abs += p * fabs(m);
  }
  u = warp_sum(u);
  mean_m = warp_sum(mean_m);
  mean_abs = warp_sum(mean_abs);

  // pass 4: central second moments
  double ve = 0.0, vm = 0.0;
  for (int i = lane; i < nc; i += 32) {
    const double m = (double)cells[i].m;
    const double e = (double)cells[i].e * scale;
    const double en = e - h * m;
    const double p = (cells[i].g * exp(-en / t - shift)) / s;
    const double de = en - u, dm = m - mean_m;
    ve += p * (de * de);
    vm += p * (dm * dm);
  }
  ve = warp_sum(ve);
  vm = warp_sum(vm);

  if (lane == 0) {
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

int launch_thermo(const unsigned long long* counts, uint32_t n_spins,
                  uint32_t n_bonds, double scale, const double* fields,
                  int n_fields, const double* temps, int n_temps, double* out,
                  void* stream) {
  const int points = n_fields * n_temps;
  if (points <= 0) return 0;
  const size_t smem = sizeof(Cell) * (size_t)(n_spins + 1) * (n_bonds + 1);
  static_assert(sizeof(Cell) * kMaxBins <= 227 * 1024, "cell list fits");
  cudaFuncSetAttribute((const void*)k2_thermo,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (points + kThermoPoints - 1) / kThermoPoints;
  k2_thermo<<<grid, kThermoThreads, smem, (cudaStream_t)stream>>>(
      counts, n_spins, n_bonds, scale, fields, temps, n_temps, points, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace isd
