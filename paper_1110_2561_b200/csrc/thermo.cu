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
// One kernel, one CTA of 256 threads per (h, T) point, straight from the
// dense table (no compaction pass: an empty bin has g = 0 and adds 0).  Warp
// w takes rows m = w, w + 8, ...; lane j takes the columns e = j + 32 c.
// The Boltzmann weight factorises over the table's axes:
//     exp(x - shift) = exp(-(E - H_min) / T) * exp(h M / T) = a_e * b_m,
// so a point needs <= 4 exponentials per lane (its columns) plus one per row
// instead of one per occupied cell; every bin then costs a few DFMAs.  The
// factors stay inside fp64 range while |h| N / T <= 300 (a_e, b_m <= e^300);
// beyond that the kernel takes one exp of the whole argument per occupied
// bin.  The product differs from exp(x - shift) by a few ulp (the GPU tests
// hold every field to 1e-12 of the reference).  Each pass ends in a fixed
// block reduction (xor-shuffle tree per warp, then the 8 warp partials in
// order), so a point's value does not depend on which other points share
// the launch (thermo_sweep(...)[0] == partition_point(...) exactly,
// test_thermo.py:85-87).
//
// (History: one CTA per point over the whole table 42 us -> warp per point
// over a per-CTA compacted cell list 33 us -> separate one-CTA compaction +
// four-warp teams 16.5 us (c5, 702 points) -> this kernel.)
#include <cuda_runtime.h>
#include <math.h>

#include <mutex>

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

__global__ void __launch_bounds__(kThermoThreads)
    k2_thermo(const unsigned long long* __restrict__ table, uint32_t n,
              uint32_t b, double scale, const double* __restrict__ fields,
              const double* __restrict__ temps, int n_temps, int n_points,
              double* __restrict__ out) {
  __shared__ double part[kThermoWarps][4];
  __shared__ double bm_s[ISD_MAX_SPINS + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int point = blockIdx.x;
  if (point >= n_points) return;  // (uniform per CTA)
  const double h = fields[point / n_temps];
  const double t = temps[point % n_temps];
  const int rows = (int)n + 1, cols = (int)b + 1;
  auto block_reduce = [&](double* v, int nv, bool is_min) {
    for (int k = 0; k < nv; ++k)
      v[k] = is_min ? warp_min(v[k]) : warp_sum(v[k]);
    if (lane == 0)
      for (int k = 0; k < nv; ++k) part[warp][k] = v[k];
    __syncthreads();
    for (int k = 0; k < nv; ++k) {
      double r = part[0][k];
#pragma unroll
      for (int w = 1; w < kThermoWarps; ++w)
        r = is_min ? fmin(r, part[w][k]) : r + part[w][k];
      v[k] = r;
    }
    __syncthreads();
  };
  auto count = [&](int r, int e) {
    return (double)__ldg(table + (size_t)r * cols + e);
  };
  double ecol[kColSlots];  // E of this lane's columns
#pragma unroll
  for (int c = 0; c < kColSlots; ++c)
    ecol[c] = (double)(2 * (lane + 32 * c) - (int)b) * scale;

  // pass 1: H_min = min over occupied bins of E - h M; shift = -H_min / T
  // (= max of x = -H / T: division by T > 0 is monotone)
  double red[4];
  red[0] = INFINITY;
  for (int r = warp; r < rows; r += kThermoWarps) {
    const double m = (double)(2 * r - (int)n);
#pragma unroll
    for (int c = 0; c < kColSlots; ++c) {
      const int e = lane + 32 * c;
      if (e < cols && count(r, e) != 0.0) red[0] = fmin(red[0], ecol[c] - h * m);
    }
  }
  block_reduce(red, 1, true);
  const double hmin = red[0];
  const double shift = -hmin / t;
  const bool split = fabs(h) * (double)n / t <= kSplitMax;
  // the factors: a_e per lane column, b_m per row (shared)
  double acol[kColSlots];
#pragma unroll
  for (int c = 0; c < kColSlots; ++c)
    acol[c] = split ? exp(-(ecol[c] - hmin) / t) : 0.0;
  if (split)
    for (int r = threadIdx.x; r < rows; r += kThermoThreads)
      bm_s[r] = exp(h * (double)(2 * r - (int)n) / t);
  __syncthreads();
  // w of bin (r, e): g a_e b_m, or (beyond the split range) one exp of the
  // whole argument for an occupied bin
  auto weight = [&](double g, int c, int r, double en) {
    if (split) return g * acol[c] * bm_s[r];
    return g != 0.0 ? g * exp(-(en - hmin) / t) : 0.0;
  };

  // pass 2: s = sum w and the first moments as w-weighted sums
  red[0] = red[1] = red[2] = red[3] = 0.0;
  for (int r = warp; r < rows; r += kThermoWarps) {
    const double m = (double)(2 * r - (int)n);
#pragma unroll
    for (int c = 0; c < kColSlots; ++c) {
      const int e = lane + 32 * c;
      if (e >= cols) continue;
      const double en = ecol[c] - h * m;
      const double w = weight(count(r, e), c, r, en);
      red[0] += w;
      red[1] += w * en;
      red[2] += w * m;
      red[3] += w * fabs(m);
    }
  }
  block_reduce(red, 4, false);
  const double s = red[0];
  const double u = red[1] / s;
  const double mean_m = red[2] / s;
  const double mean_abs = red[3] / s;

  // pass 3: central second moments (the two-pass form of thermo.py:75-77;
  // the raw <H^2> - <H>^2 form cancels catastrophically at low T)
  red[0] = red[1] = 0.0;
  for (int r = warp; r < rows; r += kThermoWarps) {
    const double m = (double)(2 * r - (int)n);
    const double dm = m - mean_m;
#pragma unroll
    for (int c = 0; c < kColSlots; ++c) {
      const int e = lane + 32 * c;
      if (e >= cols) continue;
      const double en = ecol[c] - h * m;
      const double w = weight(count(r, e), c, r, en);
      const double de = en - u;
      red[0] += w * (de * de);
      red[1] += w * (dm * dm);
    }
  }
  block_reduce(red, 2, false);
  const double ve = red[0] / s;
  const double vm = red[1] / s;

  if (threadIdx.x == 0) {
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
    k2_thermo<<<points, kThermoThreads, 0, st>>>(table, n_spins, n_bonds,
                                                 scale, fields, temps, n_temps,
                                                 points, out);
    ++launched;
  }
  cudaError_t e = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? launched : -(int)e;
}

}  // namespace isd
