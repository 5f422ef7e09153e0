// K0 — pipe-rate microbenchmarks that calibrate the integer roofline.
//
// The enumeration kernels issue POPC, LOP3, SHF, IADD3 and shared-memory
// reductions.  The per-SM issue rates of those instructions on sm_100a are
// not documented in this image, so they are measured here, on the box, with
// one CTA of 1024 threads per SM and SM clock64() bracketing a long
// unrolled loop of independent chains.  Result: lanes per clock per SM.
#include <cuda_runtime.h>

#include "isd_internal.h"

namespace isd {

constexpr int kCalThreads = 1024;
constexpr int kCalIters = 4096;
constexpr int kChains = 8;

__global__ void __launch_bounds__(kCalThreads)
    k0_cal(int which, uint32_t seed, unsigned long long* cycles,
           uint32_t* sink) {
  __shared__ uint32_t sh[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t v[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) v[i] = seed * (threadIdx.x + 7 * i + 1);
  const uint32_t a = seed ^ 0x9E3779B9u, b2 = seed * 3u + 1u;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sh);
  __syncthreads();
  const unsigned long long t0 = clock64();
  switch (which) {
    case 0:  // POPC
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i)
          asm volatile("popc.b32 %0, %0;" : "+r"(v[i]));
      }
      break;
    case 1:  // LOP3
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i)
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;"
                       : "+r"(v[i])
                       : "r"(a), "r"(b2));
      }
      break;
    case 2:  // IADD3
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i)
          asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;"
                       : "+r"(v[i])
                       : "r"(a), "r"(b2));
      }
      break;
    case 3:  // RED.shared, conflict-free (lane -> own bank)
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
          const uint32_t addr =
              sbase + 4u * (lane + 32u * ((it * kChains + i) & 255));
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        }
      }
      break;
    case 4:  // RED.shared, hashed bins over a 4033-bin table (realistic)
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
          v[i] = v[i] * 1664525u + 1013904223u;
          const uint32_t addr = sbase + 4u * ((v[i] >> 8) % 4033u);
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        }
      }
      break;
    case 5:  // IMAD
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i)
          asm volatile("mad.lo.u32 %0, %0, %1, %2;"
                       : "+r"(v[i])
                       : "r"(a), "r"(b2));
      }
      break;
    case 6:  // SHF (funnel shift)
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i)
          asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;"
                       : "+r"(v[i])
                       : "r"(a));
      }
      break;
    case 7:  // RED.shared, all 32 lanes on one word (hardware aggregation)
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
          const uint32_t addr = sbase + 4u * (32u * ((it * kChains + i) & 255));
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        }
      }
      break;
    case 8:  // RED.shared, lane pairs share a word, 16 distinct banks
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
          const uint32_t addr =
              sbase + 4u * ((lane >> 1) + 32u * ((it * kChains + i) & 255));
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        }
      }
      break;
    case 9:  // RED.shared, 4 distinct words in one bank (8 lanes each)
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
          const uint32_t addr =
              sbase + 4u * (32u * ((lane >> 3) + 4u * ((it * kChains + i) & 63)));
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        }
      }
      break;
    case 10:  // RED.shared, 8 distinct words, distinct banks, 4 lanes each
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
          const uint32_t addr =
              sbase + 4u * ((lane >> 2) * 3u + 32u * ((it * kChains + i) & 255));
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        }
      }
      break;
    case 11:  // RED.shared.add, all lanes one word, value 1 or 65536
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
          const uint32_t addr = sbase + 4u * (32u * ((it * kChains + i) & 255));
          const uint32_t val = (lane & 1) ? 65536u : 1u;
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(val)
                       : "memory");
        }
      }
      break;
    case 12:  // RED.shared.add, lane pairs per word (16 banks), values 1/65536
      for (int it = 0; it < kCalIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
          const uint32_t addr =
              sbase + 4u * ((lane >> 1) + 32u * ((it * kChains + i) & 255));
          const uint32_t val = (lane & 1) ? 65536u : 1u;
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(val)
                       : "memory");
        }
      }
      break;
    default:
      break;
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc ^= v[i];
  if (acc == 0x12345678u) sink[0] = acc + sh[threadIdx.x];
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int run_calibration(int which, int sm_count, double* lanes_per_clk_sm,
                    double* sm_mhz) {
  unsigned long long* d_cyc = nullptr;
  uint32_t* d_sink = nullptr;
  cudaError_t e = cudaMalloc(&d_cyc, sizeof(unsigned long long) * sm_count);
  if (e != cudaSuccess) return -(int)e;
  e = cudaMalloc(&d_sink, 64);
  if (e != cudaSuccess) {
    cudaFree(d_cyc);
    return -(int)e;
  }
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  // warm-up (clocks ramp) then the measured launch
  for (int rep = 0; rep < 3; ++rep)
    k0_cal<<<sm_count, kCalThreads>>>(which, 0x1234567u + rep, d_cyc, d_sink);
  cudaEventRecord(ev0);
  k0_cal<<<sm_count, kCalThreads>>>(which, 0x7654321u, d_cyc, d_sink);
  cudaEventRecord(ev1);
  e = cudaEventSynchronize(ev1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  unsigned long long* h = new unsigned long long[sm_count];
  if (e == cudaSuccess)
    e = cudaMemcpy(h, d_cyc, sizeof(unsigned long long) * sm_count,
                   cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) {
    // median per-block cycle count
    double sum = 0, mx = 0;
    for (int i = 0; i < sm_count; ++i) {
      sum += (double)h[i];
      if ((double)h[i] > mx) mx = (double)h[i];
    }
    const double cyc = sum / sm_count;
    const double ops_per_insn = (which == 2) ? 2.0 : 1.0;
    const double lanes =
        (double)kCalThreads * kCalIters * kChains * ops_per_insn;
    *lanes_per_clk_sm = lanes / cyc;
    *sm_mhz = mx / (ms * 1e3);
  }
  delete[] h;
  bump_launches(4);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaFree(d_cyc);
  cudaFree(d_sink);
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // namespace isd
