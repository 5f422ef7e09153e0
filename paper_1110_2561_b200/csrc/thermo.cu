// K2 — Z(h, T) and thermodynamics from the exact table g(M, E), fp64.
//
// Follows /root/reference/pkg/src/isingdos/thermo.py:37-88 step for step:
//   cells   = occupied (g > 0) entries, M = 2 m_idx - N, E = (2 e_idx - B)|J|
//   H       = E - h M,   x = -H / T,   shift = max over occupied cells of x
//   w       = g exp(x - shift),  s = sum w,  log Z = shift + log s,  p = w / s
//   U = p.H,  <M> = p.M,  C = p.(H-U)^2 / T^2,  chi = p.(M-<M>)^2 / T
// plus the extension <|M|> = p.|M| (BASELINE configs 2 and 5).
//
// One CTA per (h, T) point.  Each thread walks a fixed strided subset of the
// table and the partial sums are combined by a fixed shared-memory tree, so
// a point's result does not depend on which other points share the launch
// (thermo_sweep(...)[0] == partition_point(...) exactly, test_thermo.py:85-87).
#include <cuda_runtime.h>
#include <math.h>

#include "isd_internal.h"

namespace isd {

constexpr int kThermoThreads = 256;

template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red) {
  // red: K * kThermoThreads doubles
#pragma unroll
  for (int i = 0; i < K; ++i) red[i * kThermoThreads + threadIdx.x] = v[i];
  __syncthreads();
  for (int w = kThermoThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
#pragma unroll
      for (int i = 0; i < K; ++i)
        red[i * kThermoThreads + threadIdx.x] +=
            red[i * kThermoThreads + threadIdx.x + w];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = red[i * kThermoThreads];
  __syncthreads();
}

__global__ void __launch_bounds__(kThermoThreads)
    k2_thermo(const unsigned long long* __restrict__ counts, uint32_t n,
              uint32_t b, double scale, const double* __restrict__ fields,
              const double* __restrict__ temps, int n_temps,
              double* __restrict__ out) {
  __shared__ double red[3 * kThermoThreads];
  const int point = blockIdx.x;
  const double h = fields[point / n_temps];
  const double t = temps[point % n_temps];
  const uint32_t stride = b + 1;
  const uint32_t nbins = (n + 1) * stride;

  // pass 1: shift = max x over occupied cells
  double xmax = -INFINITY;
  for (uint32_t i = threadIdx.x; i < nbins; i += kThermoThreads) {
    if (counts[i] == 0) continue;
    const double m = (double)(2 * (int)(i / stride) - (int)n);
    const double e = (double)(2 * (int)(i % stride) - (int)b) * scale;
    const double en = e - h * m;
    const double x = -en / t;
    xmax = fmax(xmax, x);
  }
  red[threadIdx.x] = xmax;
  __syncthreads();
  for (int w = kThermoThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  const double shift = red[0];
  __syncthreads();

  // pass 2: s = sum g exp(x - shift)
  double v1[1] = {0.0};
  for (uint32_t i = threadIdx.x; i < nbins; i += kThermoThreads) {
    const unsigned long long g = counts[i];
    if (g == 0) continue;
    const double m = (double)(2 * (int)(i / stride) - (int)n);
    const double e = (double)(2 * (int)(i % stride) - (int)b) * scale;
    const double en = e - h * m;
    const double x = -en / t;
    v1[0] += (double)g * exp(x - shift);
  }
  block_sum<1>(v1, red);
  const double s = v1[0];

  // pass 3: first moments
  double v3[3] = {0.0, 0.0, 0.0};
  for (uint32_t i = threadIdx.x; i < nbins; i += kThermoThreads) {
    const unsigned long long g = counts[i];
    if (g == 0) continue;
    const double m = (double)(2 * (int)(i / stride) - (int)n);
    const double e = (double)(2 * (int)(i % stride) - (int)b) * scale;
    const double en = e - h * m;
    const double x = -en / t;
    const double p = ((double)g * exp(x - shift)) / s;
    v3[0] += p * en;
    v3[1] += p * m;
    v3[2] += p * fabs(m);
  }
  block_sum<3>(v3, red);
  const double u = v3[0], mean_m = v3[1], mean_abs = v3[2];

  // pass 4: central second moments
  double v2[2] = {0.0, 0.0};
  for (uint32_t i = threadIdx.x; i < nbins; i += kThermoThreads) {
    const unsigned long long g = counts[i];
    if (g == 0) continue;
    const double m = (double)(2 * (int)(i / stride) - (int)n);
    const double e = (double)(2 * (int)(i % stride) - (int)b) * scale;
    const double en = e - h * m;
    const double x = -en / t;
    const double p = ((double)g * exp(x - shift)) / s;
    const double de = en - u, dm = m - mean_m;
    v2[0] += p * (de * de);
    v2[1] += p * (dm * dm);
  }
  block_sum<2>(v2, red);

  if (threadIdx.x == 0) {
    const double log_z = shift + log(s);
    double* o = out + (size_t)point * ISD_THERMO_FIELDS;
    o[0] = log_z;
    o[1] = -t * log_z;
    o[2] = u;
    o[3] = v2[0] / (t * t);
    o[4] = mean_m;
    o[5] = v2[1] / t;
    o[6] = mean_abs;
  }
}

int launch_thermo(const unsigned long long* counts, uint32_t n_spins,
                  uint32_t n_bonds, double scale, const double* fields,
                  int n_fields, const double* temps, int n_temps, double* out,
                  void* stream) {
  const int points = n_fields * n_temps;
  if (points <= 0) return 0;
  k2_thermo<<<points, kThermoThreads, 0, (cudaStream_t)stream>>>(
      counts, n_spins, n_bonds, scale, fields, temps, n_temps, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace isd
