// K5 — the naive cross-check engine (isd_naive_enumerate).
//
// The reference keeps a deliberately plain engine next to its fast one
// (/root/reference/pkg/src/isingdos/oracle.py:71-91): decode every spin of a
// configuration from its bit, sum the spins for M, and sum S_i S_j over an
// explicit list of bonds for E.  This kernel is that engine on the GPU and
// shares nothing with K1: it takes the caller's per-slot bit positions and
// per-bond slot pairs and signs (built from the lattice geometry by
// crosscheck.py, not from the bond-class descriptor K1 runs on), evaluates
// one configuration per thread with plain loops, and counts with ordinary
// atomicAdd into its own shared table.  A fault in the bond classes, the
// hoisted decomposition or K1's histogram layout therefore shows up as a
// disagreement with this kernel (`isingdos-b200 oracle-check`).
#include <cuda_runtime.h>

#include "isd_internal.h"

namespace isd {

constexpr int kNaiveThreads = 256;
constexpr int kNaiveMaxBonds = 3 * ISD_MAX_SPINS;

struct NaiveLattice {
  uint64_t start, end;
  int32_t n_slots, n_bonds, coupling_sign;
  int32_t pad;
  uint8_t bit_of_slot[ISD_MAX_SPINS];
  uint8_t bond_i[kNaiveMaxBonds], bond_j[kNaiveMaxBonds];
  int8_t bond_sign[kNaiveMaxBonds];
};

__global__ void __launch_bounds__(kNaiveThreads)
    k5_naive(const __grid_constant__ NaiveLattice L,
             unsigned long long* __restrict__ out) {
  extern __shared__ unsigned int table[];
  const int cols = L.n_bonds + 1;
  const int bins = (L.n_slots + 1) * cols;
  for (int i = threadIdx.x; i < bins; i += blockDim.x) table[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = L.start + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
       x < L.end; x += stride) {
    int spin[ISD_MAX_SPINS];
    int m = 0;
    for (int s = 0; s < L.n_slots; ++s) {
      spin[s] = ((x >> L.bit_of_slot[s]) & 1ull) ? 1 : -1;
      m += spin[s];
    }
    int sum = 0;  // sum over bonds of sign_b S_i S_j
    for (int b = 0; b < L.n_bonds; ++b)
      sum += L.bond_sign[b] * spin[L.bond_i[b]] * spin[L.bond_j[b]];
    // E / |J| = -sign(J) sum; column (E / |J| + B) / 2, row (M + N) / 2
    const int e_col = (-L.coupling_sign * sum + L.n_bonds) / 2;
    const int m_row = (m + L.n_slots) / 2;
    atomicAdd(&table[m_row * cols + e_col], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += blockDim.x)
    if (table[i]) atomicAdd(out + i, (unsigned long long)table[i]);
}

int naive_enumerate(uint32_t n_spins, const uint32_t* bit_of_slot,
                    uint32_t n_bonds, const uint32_t* bond_slots,
                    const int32_t* bond_sign, int coupling_sign,
                    uint64_t start, uint64_t end, unsigned long long* out,
                    int sm_count, void* stream, std::string* why) {
  if (n_spins < 1 || n_spins > ISD_MAX_SPINS || n_bonds > kNaiveMaxBonds) {
    *why = "lattice outside the naive engine's limits";
    return -(int)cudaErrorInvalidValue;
  }
  NaiveLattice L{};
  L.start = start;
  L.end = end;
  L.n_slots = (int)n_spins;
  L.n_bonds = (int)n_bonds;
  L.coupling_sign = coupling_sign < 0 ? -1 : 1;
  uint64_t seen = 0;
  for (uint32_t s = 0; s < n_spins; ++s) {
    if (bit_of_slot[s] >= n_spins || ((seen >> bit_of_slot[s]) & 1)) {
      *why = "slot bit positions are not a permutation of [0, N)";
      return -(int)cudaErrorInvalidValue;
    }
    seen |= 1ull << bit_of_slot[s];
    L.bit_of_slot[s] = (uint8_t)bit_of_slot[s];
  }
  for (uint32_t b = 0; b < n_bonds; ++b) {
    if (bond_slots[2 * b] >= n_spins || bond_slots[2 * b + 1] >= n_spins ||
        (bond_sign[b] != 1 && bond_sign[b] != -1)) {
      *why = "bond slots or signs out of range";
      return -(int)cudaErrorInvalidValue;
    }
    L.bond_i[b] = (uint8_t)bond_slots[2 * b];
    L.bond_j[b] = (uint8_t)bond_slots[2 * b + 1];
    L.bond_sign[b] = (int8_t)bond_sign[b];
  }
  const size_t smem = (size_t)(n_spins + 1) * (n_bonds + 1) * 4;
  const uint64_t max_grid = (uint64_t)sm_count * 8;
  // <= 2^31 configurations per block and launch: no u32 counter can wrap
  const uint64_t per_launch = max_grid << 31;
  int launched = 0;
  for (uint64_t a = start; a < end;) {
    const uint64_t b = end - a > per_launch ? a + per_launch : end;
    L.start = a;
    L.end = b;
    const uint64_t want = (b - a + kNaiveThreads - 1) / kNaiveThreads;
    const int grid = (int)(want < max_grid ? want : max_grid);
    k5_naive<<<grid, kNaiveThreads, smem, (cudaStream_t)stream>>>(L, out);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return -(int)e;
    ++launched;
    a = b;
  }
  return launched;
}

}  // namespace isd
