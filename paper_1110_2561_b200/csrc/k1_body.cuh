// k1_body.cuh — body of the hoisted enumeration kernel (K1b).
//
// Shared, as source, by two kernels:
//   * k1_hoisted (enumerate.cu), compiled ahead of time: the lattice
//     constants come from a __grid_constant__ HoistParams (RuntimeTraits);
//   * k1_jit (jit.cpp), compiled per lattice with NVRTC: the same constants
//     are constexpr (a generated traits struct), so masks, shifts, the copy
//     offset table and the layout strides become immediates — in particular
//     each copy's constant offset folds into the RED's address immediate.
// This file must stay self-contained (builtins only): jit.cpp embeds it.
//
// Decomposition: bits [k, N) = the thread's run; inside
// [0, k) the loop sites take every subset, and 7 copy sites are 128
// register copies.  Per configuration: one add and one shared RED.

#ifndef ISD_K1_BODY_CUH
#define ISD_K1_BODY_CUH

#ifndef ISD_CHECK_ADDR
#define ISD_CHECK_ADDR(a, lo, bytes) \
  do {                               \
  } while (0)
#endif

// lane bit i of a warp flips the run bits v[i] (pivot + optional partner)
struct IsdLanes {
  unsigned long long v[5];
};

__device__ __forceinline__ void isd_red_shared_inc(unsigned int addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}

// A banded launch's work item (mirrors isd::BandItem): slots [g0, g1) of the
// free run bits in popcount order, popcounts >= q0.
struct IsdBandItem {
  unsigned long long g0, g1;
  unsigned int q0, pad;
};

// The g-th F-bit number in (popcount, value) order; *q = its popcount.
// Tables (uploaded after the launch's work items, isd::band_tables):
// cum[q] = number of F-bit values of popcount < q (q <= F + 1) and
// binom[b * (F + 1) + q] = C(b, q) for b < F, q <= F.  Warp-uniform: every
// lane walks the same slot, so the loads are broadcasts.
__device__ __forceinline__ unsigned long long isd_unrank(
    unsigned int g, int F, const unsigned int* __restrict__ cum,
    const unsigned int* __restrict__ binom, int* q) {
  int qq = 0;
  while (qq < F && g >= __ldg(cum + qq + 1)) ++qq;
  *q = qq;
  g -= __ldg(cum + qq);
  // colex rank g among the F-bit numbers of popcount qq: the highest set
  // bit is the largest b with C(b, qq) <= g, and so on down
  unsigned long long v = 0;
  for (int bit = F - 1; bit >= 0 && qq > 0; --bit) {
    const unsigned int cb = __ldg(binom + bit * (F + 1) + qq);
    if (g >= cb) {
      v |= 1ull << bit;
      g -= cb;
      --qq;
    }
  }
  return v;
}

// index of the lowest set bit (s > 0); constexpr so unrolled Gray steps fold
__host__ __device__ constexpr int isd_ctz(int s) {
  return (s & 1) ? 0 : 1 + isd_ctz(s >> 1);
}

// Gray steps S .. 2^G - 1: flip site ctz(S) to its bit in gray(S), emit.
// Each step is its own call site with constant arguments, so after inlining
// the site's constants fold (a loop here stays rolled under NVRTC).
template <int S, int G, class Flip, class Emit>
__device__ __forceinline__ void isd_gray_steps(Flip& flip, Emit& emit) {
  if constexpr (S < (1 << G)) {
    constexpr int g = isd_ctz(S);
    flip(g, (((S ^ (S >> 1)) >> g) & 1) != 0);
    emit();
    isd_gray_steps<S + 1, G>(flip, emit);
  }
}

// the next F-bit number in (popcount, value) order
__device__ __forceinline__ unsigned long long isd_next_slot(
    unsigned long long v, int F, int* q) {
  if (v != 0) {
    const unsigned long long low = v & (~v + 1);
    const unsigned long long up = v + low;
    const unsigned long long nv =
        (((up ^ v) >> 2) >> (__ffsll((long long)low) - 1)) | up;
    if (!(nv >> F)) return nv;  // same popcount
  }
  *q += 1;  // first (smallest) number of the next popcount class
  return (1ull << *q) - 1;
}

// word of bin (m, e) in the unpaired layout
template <class T>
__device__ __forceinline__ unsigned int isd_bin_word(const T& L, unsigned int m,
                                                     unsigned int e) {
  if (L.e_mode()) {
    const unsigned int par = e & 1u;
    return m * L.row_words() + ((e - par) >> 1) * L.e_words() +
           par * L.plane_words();
  }
  return m * L.row_words() + e * L.e_words();
}

// PAIR 1: copy bit 6 is not unrolled; one RED counts the configuration
// with that site down and its partner with it up, in pattern plane p (= the
// site's unsatisfied bonds while down), and the flush credits the partner
// to (m + 1, e + D - 2p).  PAIR 2: copy bit 5 as well (4 configurations per
// RED, planes p0 (bit 6) x p1 (bit 5)).
//
// Banded tables (L.band_rows() > 0, mode 2): the table holds band_rows rows
// of m relative to a work item's base row; the launch walks work items
// (slots of the free run bits in popcount order, `items`), each zeroed,
// walked and flushed in turn.
template <int NC, bool DOUBLE, int PAIR, class T>
__device__ __forceinline__ void k1_hoisted_body(
    const T& L, unsigned long long run_begin, unsigned long long nruns,
    unsigned long long hi_step, unsigned long long lane_mask,
    const IsdLanes lanes, const IsdBandItem* __restrict__ items,
    unsigned int n_items, int free_bits, unsigned int* hist,
    unsigned long long* __restrict__ out) {
  auto zero_hist = [&]() {
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    const unsigned int n4 = L.n_hist() * L.hist_words() / 4;
    for (unsigned int i = threadIdx.x; i < n4; i += blockDim.x)
      h4[i] = make_uint4(0, 0, 0, 0);
  };
  const unsigned int warp = threadIdx.x >> 5;
  const unsigned int hbase = (unsigned int)__cvta_generic_to_shared(
      hist + (warp % L.n_hist()) * L.hist_words());
  const unsigned int hbytes = 4u * L.hist_words();
  const unsigned long long gstride = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned int nloop = L.nloop();
  const unsigned long long above_k = L.above_k();
  // this lane's run-bit pattern: XOR of the vectors of its set lane bits
  unsigned long long lane_dep = 0;
  {
    const unsigned int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < 5; ++i)
      if ((lane >> i) & 1) lane_dep ^= lanes.v[i];
  }

  // slot (warp-uniform run bits) -> run: insert a 0 at each lane pivot,
  // then XOR in the lane's pattern
  auto slot_run = [&](unsigned long long hi) {
    unsigned long long m = lane_mask;
#pragma unroll
    for (int i = 0; i < 5; ++i) {  // insert a 0 at each lane bit
      const unsigned long long low = m & (~m + 1);
      hi = ((hi & ~(low - 1)) << 1) | (hi & (low - 1));
      m ^= low;
    }
    return run_begin + (hi ^ lane_dep);
  };
  // ---- one run: bits [k, N) fixed; table rows are m - row_off ----
  auto run_body = [&](unsigned long long r, unsigned int row_off) {
    // ---- per-run constants (bits [k, N) fixed) ----
    const unsigned long long xt = r << L.k();
    const int m_run = __popcll(xt);
    int e_run = 0;
    unsigned int cst[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const unsigned long long sh = xt >> L.shift(c);
      e_run += __popcll(((xt ^ sh) ^ L.jneg(c)) & L.mask(c) & above_k);
      // partner word seen by the loop sites; jneg folded in
      cst[c] = (unsigned int)sh ^ (unsigned int)L.jneg(c);
    }
    int npr[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      npr[q] = __popcll((xt ^ L.jn1(q)) & L.nm1(q) & above_k);
      if (DOUBLE) npr[q] += __popcll((xt ^ L.jn2(q)) & L.nm2(q) & above_k);
    }
    // byte address of (m_run, e = 0); the e parity of the configurations
    // is par_run ^ parity(loop bits & odd_mask)
    const unsigned int a_run =
        hbase + (unsigned int)(m_run - (int)row_off) * L.row_bytes();
    const unsigned int par_run =
        (unsigned int)(__popcll(xt & L.odd_mask()) + L.e_parity()) & 1u;
    const unsigned int odd_loop =
        (unsigned int)L.odd_mask() & L.loop_mask();
    // Gray sites (JIT builds): the G lowest loop sites are walked in Gray
    // order inside one iteration, each step one site flip updated from its
    // neighbours; their run-site partners are counted once per run
    constexpr int G = T::gray();
    int gpr[G > 0 ? G : 1];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      gpr[g] = __popcll((xt ^ L.g_jn1(g)) & L.g_nm1(g) & above_k);
      if (DOUBLE) gpr[g] += __popcll((xt ^ L.g_jn2(g)) & L.g_nm2(g) & above_k);
    }
    // ---- loop over the subsets of the loop sites ----
    const unsigned int outer = L.loop_mask() & ~L.g_mask();
    unsigned int jb = 0;
    for (unsigned int it = 0; it < (nloop >> G); ++it) {
      int e = e_run;
#pragma unroll
      for (int c = 0; c < NC; ++c)
        e += __popc((jb ^ __funnelshift_rc(jb, 0u, L.shift(c)) ^ cst[c]) &
                    L.mvar(c));
      unsigned int d[7];
      unsigned int pair_off = 0;
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        int nq = npr[q] + __popc((jb ^ L.jn1v(q)) & L.nm1v(q));
        if (DOUBLE) nq += __popc((jb ^ L.jn2v(q)) & L.nm2v(q));
        e += nq;
        d[q] = (unsigned int)((int)L.e_bytes() * (L.degree(q) - 2 * nq));
        if (PAIR >= 1 && q == 6) pair_off += (unsigned int)nq * L.pair_bytes(0);
        if (PAIR >= 2 && q == 5) pair_off += (unsigned int)nq * L.pair_bytes(1);
      }
      unsigned int par = (par_run + __popc(jb & odd_loop)) & 1u;
      // a[c] carries no per-copy constant: addr(c) = a[c] + koff(c), where
      // koff(c) = popc(c) row_bytes + e_bytes * (copy-copy unsatisfied
      // bonds of c) folds into the RED's address offset.  128 copies: a
      // 32-leaf subset-sum tree over copy bits 0-4 (live set <= 16), each
      // leaf spawning its siblings in bits 5 and 6 (paired bits: none).
      auto emit = [&]() {
        const unsigned int a0 = a_run + (unsigned int)__popc(jb) * L.row_bytes() +
                                (unsigned int)e * L.e_bytes() +
                                par * (unsigned int)L.plane_bytes() + pair_off;
        unsigned int a[32];
#pragma unroll
        for (int cl = 0; cl < 32; ++cl) {
          if (cl == 0) {
            a[0] = a0;
          } else {
            const int top = 31 - __clz(cl);
            a[cl] = a[cl ^ (1 << top)] + d[top];
          }
          ISD_CHECK_ADDR(a[cl] + L.koff(cl), hbase, hbytes);
          isd_red_shared_inc(a[cl] + L.koff(cl));
          const unsigned int b1 = a[cl] + d[5];
          if (PAIR <= 1) {
            ISD_CHECK_ADDR(b1 + L.koff(cl + 32), hbase, hbytes);
            isd_red_shared_inc(b1 + L.koff(cl + 32));
          }
          if (PAIR == 0) {
            const unsigned int b2 = a[cl] + d[6];
            const unsigned int b3 = b1 + d[6];
            ISD_CHECK_ADDR(b2 + L.koff(cl + 64), hbase, hbytes);
            isd_red_shared_inc(b2 + L.koff(cl + 64));
            ISD_CHECK_ADDR(b3 + L.koff(cl + 96), hbase, hbytes);
            isd_red_shared_inc(b3 + L.koff(cl + 96));
          }
        }
      };
      // flip Gray site g (up or down) in the current subset: its bonds to
      // non-copy sites change e by +-(D_g - 2 n_g), n_g from the current
      // neighbours; its bonds to copy sites shift those sites' unsatisfied
      // counts by the per-lattice g_cdelta (and e, d, the pattern planes)
      auto flip = [&](const int g, const bool up) {
        int ng = gpr[g] + __popc((jb ^ L.g_jn1v(g)) & L.g_nm1v(g));
        if (DOUBLE) ng += __popc((jb ^ L.g_jn2v(g)) & L.g_nm2v(g));
        const int sg = up ? 1 : -1;
        e += sg * (L.g_deg(g) - 2 * ng + L.g_csum(g));
#pragma unroll
        for (int q = 0; q < 7; ++q)
          if (L.g_cdelta(g, q) != 0) {
            d[q] -= (unsigned int)(sg * 2 * (int)L.e_bytes() * L.g_cdelta(g, q));
            if (PAIR >= 1 && q == 6)
              pair_off += (unsigned int)(sg * L.g_cdelta(g, q) *
                                         (int)L.pair_bytes(0));
            if (PAIR >= 2 && q == 5)
              pair_off += (unsigned int)(sg * L.g_cdelta(g, q) *
                                         (int)L.pair_bytes(1));
          }
        if (L.g_odd(g)) par ^= 1u;
        jb ^= L.g_bit(g);
      };
      // the 2^G subsets of the Gray sites in reflected Gray-code order:
      // step s flips site ctz(s), to its value in gray(s) = s ^ (s >> 1)
      // (unrolled at compile time, so every site index is a constant)
      emit();
      isd_gray_steps<1, G>(flip, emit);
      jb = ((jb & outer) - outer) & outer;  // next subset (Gray sites clear)
    }
  };
  // ---- flush: table rows [0, rows) at absolute row row_off -> bins ----
  auto flush = [&](unsigned int row_off, unsigned int rows) {
    const unsigned int m_lo = row_off;
    unsigned int m_hi = row_off + rows + (PAIR > 0 ? PAIR : 0);  // exclusive
    if (m_hi > L.nbins() / L.stride()) m_hi = L.nbins() / L.stride();
    // single parity plane: bins of the other parity are always 0 (and their
    // words alias), so only the bins of parity e_parity are visited
    const bool one_plane = L.e_mode() && L.odd_mask() == 0;
    const unsigned int e0 = one_plane ? (unsigned int)L.e_parity() : 0u;
    const unsigned int e_step = one_plane ? 2u : 1u;
    const unsigned int per_row = (L.stride() - e0 + e_step - 1) / e_step;
    const unsigned int n_units = (m_hi - m_lo) * per_row;
    for (unsigned int u = threadIdx.x; u < n_units; u += blockDim.x) {
      const unsigned int mr = u / per_row;
      const unsigned int m = m_lo + mr;
      const unsigned int e = e0 + (u - mr * per_row) * e_step;
      const unsigned int bin = m * L.stride() + e;
      const int row = (int)(m - row_off);  // table row of this bin
      // words are linear in the row and, for the even shifts the pairing
      // makes, in e: word(r - dr, e - de) = word(r, e) - dr A - de_words(de)
      const int gw = (int)isd_bin_word(L, 0u, e);
      auto de_words = [&](int de) {
        return L.e_mode() ? (de >> 1) * (int)L.e_words() : de * (int)L.e_words();
      };
      auto row_ok = [&](int r) { return r >= 0 && r < (int)rows; };
      auto e_ok = [&](int ee) { return ee >= 0 && ee < (int)L.stride(); };
      const int A = (int)L.row_words();
      unsigned long long s = 0;
      for (unsigned int h = 0; h < L.n_hist(); ++h) {
        const unsigned int* hh = hist + h * L.hist_words();
        if constexpr (PAIR == 0) {
          if (row_ok(row)) s += hh[row * A + gw];
        } else if constexpr (PAIR == 1) {
          const int D0 = L.pair_deg(0);
          const bool ok0 = row_ok(row), ok1 = row_ok(row - 1);
          const int w0 = row * A + gw, w1 = w0 - A;
#pragma unroll
          for (int p = 0; p <= D0; ++p) {
            const int plane = p * (int)L.pair_words(0);
            const int f = D0 - 2 * p;
            if (ok0) s += hh[w0 + plane];  // paired site down
            if (ok1 && e_ok((int)e - f))   // ... up: the partner
              s += hh[w1 + plane - de_words(f)];
          }
        } else {
          const int D0 = L.pair_deg(0), D1 = L.pair_deg(1);
          const bool ok0 = row_ok(row), ok1 = row_ok(row - 1),
                     ok2 = row_ok(row - 2);
          const int w0 = row * A + gw, w1 = w0 - A, w2 = w0 - 2 * A;
#pragma unroll
          for (int p1 = 0; p1 <= D1; ++p1)
#pragma unroll
            for (int p0 = 0; p0 <= D0; ++p0) {
              const int plane = p0 * (int)L.pair_words(0) +
                                p1 * (int)L.pair_words(1);
              const int f0 = D0 - 2 * p0, f1 = D1 - 2 * p1;
              const int f2 = f0 + f1 + L.pair_both();
              if (ok0) s += hh[w0 + plane];  // both paired sites down
              if (ok1 && e_ok((int)e - f0))  // bit-6 site up
                s += hh[w1 + plane - de_words(f0)];
              if (ok1 && e_ok((int)e - f1))  // bit-5 site up
                s += hh[w1 + plane - de_words(f1)];
              if (ok2 && e_ok((int)e - f2))  // both up
                s += hh[w2 + plane - de_words(f2)];
            }
        }
      }
      if (s) atomicAdd(out + bin, s);
    }
  };

  if (L.band_rows() == 0) {
    // ---- grid-stride walk over the runs; one table for all rows ----
    zero_hist();
    __syncthreads();
    for (unsigned long long t =
             (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
         t < nruns; t += gstride) {
      // The 32 lanes of a warp differ by XORs of five run-bit vectors, each
      // with its own pivot bit (lane_mask): which sites they differ in sets
      // the shared-memory bank spread.  The warp's slot spreads over the
      // non-pivot run bits, so (slot, lane) -> run is a bijection.  Warp w
      // takes slot w * hi_step (1 in a walk; > 1 when the autotuner times a
      // sample of warps spread over the whole range).
      run_body(slot_run((t >> 5) * hi_step), 0u);
    }
    __syncthreads();
    flush(0u, L.nbins() / L.stride());
  } else {
    // ---- banded: work items of slots in popcount order ----
    const unsigned int warps = blockDim.x >> 5;
    const unsigned int lane = threadIdx.x & 31;
    const unsigned int base_popc =
        (unsigned int)__popcll(run_begin << L.k());
    const unsigned int* cum =
        reinterpret_cast<const unsigned int*>(items + n_items);
    const unsigned int* binom = cum + free_bits + 2;
    __shared__ unsigned int next_slot;  // the item's first unclaimed slot
    for (unsigned int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const IsdBandItem item = items[it];
      zero_hist();
      if (threadIdx.x == 0) next_slot = 0;
      __syncthreads();
      const unsigned int row_off = base_popc + item.q0;
      // Warps claim chunks of the item's slots (guided: a chunk is 1/(2W)
      // of what is left, down to one slot), so they finish within about
      // one slot of each other; each chunk starts with a table unrank and
      // steps in popcount order.
      const unsigned int n_slots = (unsigned int)(item.g1 - item.g0);
      for (;;) {
        unsigned int start = 0, cnt = 0;
        if (lane == 0) {
          unsigned int old = *(volatile unsigned int*)&next_slot;
          while (old < n_slots) {
            cnt = (n_slots - old) / (2u * warps);
            if (cnt == 0) cnt = 1;
            const unsigned int seen = atomicCAS(&next_slot, old, old + cnt);
            if (seen == old) break;
            old = seen;
            cnt = 0;
          }
          start = old;
        }
        cnt = __shfl_sync(0xffffffffu, cnt, 0);
        if (cnt == 0) break;
        start = __shfl_sync(0xffffffffu, start, 0);
        int q = 0;
        unsigned long long v = isd_unrank((unsigned int)item.g0 + start,
                                          free_bits, cum, binom, &q);
        for (unsigned int i = 0; i < cnt; ++i) {
          run_body(slot_run(v), row_off);
          v = isd_next_slot(v, free_bits, &q);
        }
      }
      __syncthreads();
      flush(row_off, L.band_rows());
      __syncthreads();
    }
  }
}

#endif  // ISD_K1_BODY_CUH
