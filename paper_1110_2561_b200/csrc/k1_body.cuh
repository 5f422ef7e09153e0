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
// free run bits in popcount order, popcounts >= q0; mirror != 0: the item's
// table holds its rows in descending order.
struct IsdBandItem {
  unsigned long long g0, g1;
  unsigned int q0, mirror;
};

// A banded launch's slot -> run-bit map: free bit i of a slot (the i-th bit
// of its popcount-ordered value) lands on run bit pos(i), given as up to 16
// fields of consecutive bits that move together: run bits of the slot =
// OR_j rotl32(v & mask[j], rot[j]).  The natural order (i-th lowest
// non-pivot run bit) is one such map; the host may instead put the run
// sites that decide an item's bank conflicts on top of the order, so that
// the slots of an item agree on them (capi.cu band_slot_order).
struct IsdSlotMap {
  unsigned int mask[16];
  unsigned int rot[16];
};

// The layout of a mirrored work item: row r of the band lives at row
// band_rows - 1 - r, i.e. the row stride is -A from an origin at the last
// row.  Which banks the 32 lanes' words fall on depends on the sign of the
// row stride (word = +-m A + e' + plane S): the descending order gives a
// popcount class the conflicts its mirror image has in ascending order, so
// the host picks per item whichever its cost model scores lower.
template <class T>
struct IsdMirror : T {
  __device__ __forceinline__ explicit IsdMirror(const T& t) : T(t) {}
  __device__ __forceinline__ unsigned int row_bytes() const {
    return 0u - T::row_bytes();
  }
  __device__ __forceinline__ unsigned int row_words() const {
    return 0u - T::row_words();
  }
  // copy c's offset holds popc(c) row steps
  __device__ __forceinline__ unsigned int koff(int c) const {
    return T::koff(c) - 2u * (unsigned int)__popc((unsigned int)c) * T::row_bytes();
  }
};
template <class T>
__device__ __forceinline__ unsigned int isd_row_origin(const T&) {
  return 0u;
}
template <class T>
__device__ __forceinline__ unsigned int isd_row_origin(const IsdMirror<T>& M) {
  return (M.band_rows() - 1u) * M.T::row_words();
}

// Binomial coefficients C(n, k), n, k < 24, in constant memory: the unrank
// below reads them with warp-uniform indices (constant-cache broadcasts).
struct IsdBinom {
  unsigned int c[24][24];
};
__host__ __device__ constexpr IsdBinom isd_make_binom() {
  IsdBinom b{};
  for (int n = 0; n < 24; ++n)
    for (int k = 0; k < 24; ++k)
      b.c[n][k] = k == 0 ? 1u : (n == 0 ? 0u : b.c[n - 1][k - 1] + b.c[n - 1][k]);
  return b;
}
__constant__ IsdBinom isd_binom = isd_make_binom();

// The g-th F-bit number in (popcount, value) order; *q = its popcount
// (F <= 23, checked by the host).  Warp-uniform.
__device__ __forceinline__ unsigned long long isd_unrank(unsigned int g, int F,
                                                         int* q) {
  int qq = 0;
  while (qq < F && g >= isd_binom.c[F][qq]) g -= isd_binom.c[F][qq++];
  *q = qq;
  // colex rank g among the F-bit numbers of popcount qq: the highest set
  // bit is the largest b with C(b, qq) <= g, and so on down
  unsigned long long v = 0;
  for (int bit = F - 1; bit >= 0 && qq > 0; --bit) {
    const unsigned int cb = isd_binom.c[bit][qq];
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

// Index of the multiset {a, b, c} (values 0..R) in (largest, middle,
// smallest) order: C(hi + 2, 3) + C(mid + 1, 2) + lo (plan.cpp tri_index).
__device__ __forceinline__ unsigned int isd_tri_index(int a, int b, int c) {
  const int lo = min(a, min(b, c)), hi = max(a, max(b, c));
  const int mid = a + b + c - lo - hi;
  return (unsigned int)(hi * (hi + 1) * (hi + 2) / 6 + ((mid * (mid + 1)) >> 1) +
                        lo);
}

// PAIR 1: copy bit 6 is not unrolled; one RED counts the configuration
// with that site down and its partner with it up, in pattern plane p (= the
// site's unsatisfied bonds while down), and the flush credits the partner
// to (m + 1, e + D - 2p).  PAIR 2: copy bit 5 as well (4 configurations per
// RED, planes p0 (bit 6) x p1 (bit 5)).  PAIR 3: copy bits 4, 5, 6 are a
// cluster of three like sites (equal degree, pairwise joined alike, no bond
// to the unpaired copy sites): one RED counts the cluster's 8
// configurations, in the plane of the multiset of the three sites'
// unsatisfied external bonds; the flush credits the subset U flipped up to
// (m + |U|, e + sum_U (R - 2 n_i) + [|U| = 1 or 2] pair_both).
//
// Banded tables (L.band_rows() > 0, modes 2 and 3): the table holds
// band_rows rows of m relative to a work item's base row; the launch walks
// work items (slots of the free run bits in popcount order, `items`), each
// zeroed, walked and flushed in turn.  A slot's bits reach their run bits
// through `smap`; an item marked `mirror` keeps its rows in descending
// order (IsdMirror); `item_clk`, when given, receives every item's SM
// cycles (the host's calibration launch).
template <int NC, bool DOUBLE, int PAIR, class T>
__device__ __forceinline__ void k1_hoisted_body(
    const T& L, unsigned long long run_begin, unsigned long long nruns,
    unsigned long long hi_step, unsigned long long lane_mask,
    const IsdLanes lanes, const IsdBandItem* __restrict__ items,
    unsigned int n_items, int free_bits, unsigned int* claim,
    const IsdSlotMap& smap, unsigned long long* item_clk, unsigned int* hist,
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
  // banded launches: the slot's bits through the launch's slot map
  auto band_run = [&](unsigned long long v) {
    const unsigned int x = (unsigned int)v;
    unsigned int r = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      r |= __funnelshift_l(x & smap.mask[j], x & smap.mask[j], smap.rot[j]);
    return run_begin + ((unsigned long long)r ^ lane_dep);
  };
  // ---- one run: bits [k, N) fixed; table rows are m - row_off ----
  auto run_body = [&](const auto& L, unsigned long long r,
                      unsigned int row_off) {
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
        hbase + 4u * isd_row_origin(L) +
        (unsigned int)(m_run - (int)row_off) * L.row_bytes();
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
      int pn[3] = {0, 0, 0};  // PAIR 3: the cluster sites' unsatisfied bonds
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        int nq = npr[q] + __popc((jb ^ L.jn1v(q)) & L.nm1v(q));
        if (DOUBLE) nq += __popc((jb ^ L.jn2v(q)) & L.nm2v(q));
        e += nq;
        d[q] = (unsigned int)((int)L.e_bytes() * (L.degree(q) - 2 * nq));
        if (PAIR == 3) {
          if (q >= 4) pn[q - 4] = nq;
        } else {
          if (PAIR >= 1 && q == 6) pair_off += (unsigned int)nq * L.pair_bytes(0);
          if (PAIR >= 2 && q == 5) pair_off += (unsigned int)nq * L.pair_bytes(1);
        }
      }
      if (PAIR == 3)
        pair_off = isd_tri_index(pn[0], pn[1], pn[2]) * L.pair_bytes(0);
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
        constexpr int kTree = PAIR == 3 ? 16 : 32;
        unsigned int a[kTree];
#pragma unroll
        for (int cl = 0; cl < kTree; ++cl) {
          if (cl == 0) {
            a[0] = a0;
          } else {
            const int top = 31 - __clz(cl);
            a[cl] = a[cl ^ (1 << top)] + d[top];
          }
          ISD_CHECK_ADDR(a[cl] + L.koff(cl), hbase, hbytes);
          isd_red_shared_inc(a[cl] + L.koff(cl));
          if (PAIR == 3) continue;
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
        bool touched = false;  // PAIR 3: a cluster site's count changed
#pragma unroll
        for (int q = 0; q < 7; ++q)
          if (L.g_cdelta(g, q) != 0) {
            d[q] -= (unsigned int)(sg * 2 * (int)L.e_bytes() * L.g_cdelta(g, q));
            if (PAIR == 3) {
              if (q >= 4) {
                pn[q - 4] += sg * L.g_cdelta(g, q);
                touched = true;
              }
              continue;
            }
            if (PAIR >= 1 && q == 6)
              pair_off += (unsigned int)(sg * L.g_cdelta(g, q) *
                                         (int)L.pair_bytes(0));
            if (PAIR >= 2 && q == 5)
              pair_off += (unsigned int)(sg * L.g_cdelta(g, q) *
                                         (int)L.pair_bytes(1));
          }
        if (PAIR == 3 && touched)
          pair_off = isd_tri_index(pn[0], pn[1], pn[2]) * L.pair_bytes(0);
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
#ifdef ISD_PROBE
  long long probe_t1 = 0;  // (probe build) end of the flush's stage 1
#endif
  auto flush = [&](const auto& L, unsigned int row_off, unsigned int rows) {
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
    // words are linear in the row and, for the even shifts the pairing
    // makes, in e: word(r - dr, e - de) = word(r, e) - dr A - de_words(de)
    auto de_words = [&](int de) {
      return L.e_mode() ? (de >> 1) * (int)L.e_words() : de * (int)L.e_words();
    };
    auto row_ok = [&](int r) { return r >= 0 && r < (int)rows; };
    auto e_ok = [&](int ee) { return ee >= 0 && ee < (int)L.stride(); };
    const int A = (int)L.row_words();
    const int org = (int)isd_row_origin(L);  // word of row 0
    if constexpr (PAIR == 2) {
      // Separable two-stage flush.  A bin (m, e) collects, over the pattern
      // planes (p0, p1), its own word and its three partners':
      //   H[r, e] + H[r-1, e-f0] + H[r-1, e-f1] + H[r-2, e-f0-f1-t]
      // (r = m - row_off, f_i = D_i - 2 p_i).  Stage 1 folds p0 per
      // (r, e, p1): X = sum_p0 H[r, e], Y = sum_p0 H[r, e - f0], written in
      // place over the words of p0 = 0 and 1 (a warp owns a whole (r, p1)
      // slice, so only the warp syncs); stage 2 then needs 4 words per p1:
      //   X[r, e] + Y[r-1, e] + X[r-1, e-f1] + Y[r-2, e-f1-t].
      // 14 (D0 + 1) + 4 (D1 + 1) words per bin instead of 4 (D0+1)(D1+1).
      const int D0 = L.pair_deg(0), D1 = L.pair_deg(1);
      const int S0 = (int)L.pair_words(0), S1 = (int)L.pair_words(1);
      const int y_off = D0 >= 1 ? S0 : 0;  // D0 = 0: Y = X
      const unsigned int lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
      const unsigned int slices = rows * (unsigned int)(D1 + 1);
      constexpr int kE = 4;  // e units per lane (per_row <= 128)
      for (unsigned int g = warp; g < slices * L.n_hist(); g += nwarps) {
        unsigned int* hh = hist + (g / slices) * L.hist_words();
        const unsigned int sl = g % slices;
        const int r = (int)(sl / (unsigned int)(D1 + 1));
        const int p1 = (int)(sl % (unsigned int)(D1 + 1));
        unsigned int xs[kE], ys[kE];
        int base[kE];
#pragma unroll
        for (int j = 0; j < kE; ++j) {
          const unsigned int u = lane + 32u * j;
          xs[j] = ys[j] = 0u;
          base[j] = 0;
          if (u < per_row) {
            const unsigned int e = e0 + u * e_step;
            base[j] = org + r * A + (int)isd_bin_word(L, 0u, e) + p1 * S1;
#pragma unroll
            for (int p0 = 0; p0 <= D0; ++p0) {
              const int f0 = D0 - 2 * p0;
              xs[j] += hh[base[j] + p0 * S0];
              if (e_ok((int)e - f0)) ys[j] += hh[base[j] + p0 * S0 - de_words(f0)];
            }
          }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kE; ++j)
          if (lane + 32u * j < per_row) {
            hh[base[j]] = xs[j];
            hh[base[j] + y_off] = ys[j];
          }
        __syncwarp();
      }
      __syncthreads();
#ifdef ISD_PROBE
      probe_t1 = clock64();
#endif
      // (each block starts at its own offset: blocks flushing at the same
      // time then add into different lines of the global table)
      const unsigned int rot = (blockIdx.x * 97u) % n_units;
      for (unsigned int v = threadIdx.x; v < n_units; v += blockDim.x) {
        const unsigned int u = v + rot < n_units ? v + rot : v + rot - n_units;
        const unsigned int mr = u / per_row;
        const unsigned int m = m_lo + mr;
        const unsigned int e = e0 + (u - mr * per_row) * e_step;
        const int row = (int)(m - row_off);
        const int gw = (int)isd_bin_word(L, 0u, e);
        const bool ok0 = row_ok(row), ok1 = row_ok(row - 1),
                   ok2 = row_ok(row - 2);
        unsigned long long s = 0;
        for (unsigned int h = 0; h < L.n_hist(); ++h) {
          const unsigned int* hh = hist + h * L.hist_words();
          unsigned int s32 = 0;  // < 2^32: an item holds < 2^32 configurations
#pragma unroll
          for (int p1 = 0; p1 <= D1; ++p1) {
            const int f1 = D1 - 2 * p1, ft = f1 + L.pair_both();
            const int w0 = org + row * A + gw + p1 * S1;
            if (ok0) s32 += hh[w0];                             // X[r, e]
            if (ok1) s32 += hh[w0 - A + y_off];                 // Y[r-1, e]
            if (ok1 && e_ok((int)e - f1))
              s32 += hh[w0 - A - de_words(f1)];                 // X[r-1, e-f1]
            if (ok2 && e_ok((int)e - ft))
              s32 += hh[w0 - 2 * A - de_words(ft) + y_off];     // Y[r-2, ..]
          }
          s += s32;
        }
        if (s) atomicAdd(out + m * L.stride() + e, s);
      }
    } else if constexpr (PAIR == 3) {
      // A bin (m, e) collects, over the multiset planes {a <= b <= c} and the
      // subsets U of the cluster flipped up, H[r - |U|, e - de(U), plane],
      // de(U) = sum_U (R - 2 n_i) + [|U| = 1 or 2] I1.
      const int R = L.pair_deg(0), I1 = L.pair_both();
      const int S = (int)L.pair_words(0);
      const unsigned int rot = (blockIdx.x * 97u) % n_units;
      // Specialised build with at least as many planes as folded sums
      // (R >= 4): a two-stage flush.  The shift a flipped subset U applies
      // depends on the plane {a, b, c} only through a symmetric function of
      // it — the value of the one site up, the sum of the two, the sum of
      // all three — so stage 1 folds the planes of every table cell into
      //   G0 = sum_p H_p,   G1[v] = sum_p #{i : p_i = v} H_p,
      //   G2[t] = sum_p #{i < j : p_i + p_j = t} H_p,
      //   G3[t] = sum_{p : a + b + c = t} H_p
      // (6R + 4 sums, written in place over the cell's first planes; a
      // thread owns its cell, the block syncs once), and stage 2 reads
      //   G0[r, e] + sum_v G1[v][r-1, e - (R-2v) - I1]
      //            + sum_t G2[t][r-2, e - (2R-2t) - I1]
      //            + sum_t G3[t][r-3, e - (3R-2t)]:
      // planes + 2 (6R + 4) shared accesses per cell instead of 8 x planes.
      constexpr int kR = T::tri_r();
      constexpr int kNP = kR < 0 ? 0 : (kR + 1) * (kR + 2) * (kR + 3) / 6;
      constexpr int kNG = 6 * kR + 4;
      if constexpr (kR >= 0 && kNG <= kNP) {
        const unsigned int n_cells = rows * per_row;
        for (unsigned int h = 0; h < L.n_hist(); ++h) {
          unsigned int* hh0 = hist + h * L.hist_words();
          for (unsigned int v = threadIdx.x; v < n_cells; v += blockDim.x) {
            const unsigned int r = v / per_row;
            const unsigned int e = e0 + (v - r * per_row) * e_step;
            unsigned int* hh = hh0 + org + (int)r * A + (int)isd_bin_word(L, 0u, e);
            unsigned int g0 = 0, g1[kR + 1] = {}, g2[2 * kR + 1] = {},
                         g3[3 * kR + 1] = {};
#pragma unroll
            for (int c = 0; c <= kR; ++c)
#pragma unroll
              for (int b = 0; b <= c; ++b)
#pragma unroll
                for (int a = 0; a <= b; ++a) {
                  const unsigned int x =
                      hh[(c * (c + 1) * (c + 2) / 6 + b * (b + 1) / 2 + a) * S];
                  g0 += x;
                  g1[a] += x;
                  g1[b] += x;
                  g1[c] += x;
                  g2[a + b] += x;
                  g2[a + c] += x;
                  g2[b + c] += x;
                  g3[a + b + c] += x;
                }
            hh[0] = g0;
#pragma unroll
            for (int i = 0; i <= kR; ++i) hh[(1 + i) * S] = g1[i];
#pragma unroll
            for (int i = 0; i <= 2 * kR; ++i) hh[(kR + 2 + i) * S] = g2[i];
#pragma unroll
            for (int i = 0; i <= 3 * kR; ++i) hh[(3 * kR + 3 + i) * S] = g3[i];
          }
        }
        __syncthreads();
        for (unsigned int v = threadIdx.x; v < n_units; v += blockDim.x) {
          const unsigned int u = v + rot < n_units ? v + rot : v + rot - n_units;
          const unsigned int mr = u / per_row;
          const unsigned int m = m_lo + mr;
          const unsigned int e = e0 + (u - mr * per_row) * e_step;
          const int row = (int)(m - row_off);
          const int gw = (int)isd_bin_word(L, 0u, e);
          unsigned long long s = 0;
          for (unsigned int h = 0; h < L.n_hist(); ++h) {
            const unsigned int* hh =
                hist + h * L.hist_words() + org + row * A + gw;
            unsigned int s32 = 0;  // (multiplicities <= 3: still < 2^32)
            auto term = [&](int dr, int de, int j) {
              if (e_ok((int)e - de)) s32 += hh[j * S - dr * A - de_words(de)];
            };
            if (row_ok(row)) s32 += hh[0];
            if (row_ok(row - 1)) {
#pragma unroll
              for (int i = 0; i <= kR; ++i) term(1, kR - 2 * i + I1, 1 + i);
            }
            if (row_ok(row - 2)) {
#pragma unroll
              for (int i = 0; i <= 2 * kR; ++i)
                term(2, 2 * kR - 2 * i + I1, kR + 2 + i);
            }
            if (row_ok(row - 3)) {
#pragma unroll
              for (int i = 0; i <= 3 * kR; ++i)
                term(3, 3 * kR - 2 * i, 3 * kR + 3 + i);
            }
            s += s32;
          }
          if (s) atomicAdd(out + m * L.stride() + e, s);
        }
        return;
      }
      for (unsigned int v = threadIdx.x; v < n_units; v += blockDim.x) {
        const unsigned int u = v + rot < n_units ? v + rot : v + rot - n_units;
        const unsigned int mr = u / per_row;
        const unsigned int m = m_lo + mr;
        const unsigned int e = e0 + (u - mr * per_row) * e_step;
        const int row = (int)(m - row_off);
        const int gw = (int)isd_bin_word(L, 0u, e);
        const bool ok0 = row_ok(row), ok1 = row_ok(row - 1),
                   ok2 = row_ok(row - 2), ok3 = row_ok(row - 3);
        unsigned long long s = 0;
        // One sweep over the planes per number of sites flipped up, the row
        // test outside it.  In the specialised build R is a constant and
        // the sweeps unroll: every plane offset and energy shift is then an
        // immediate, a term costs its range test, a load and an add.
        // term(dr, de, word): H[row - dr, e - de, plane at word offset]
        for (unsigned int h = 0; h < L.n_hist(); ++h) {
          const unsigned int* hh =
              hist + h * L.hist_words() + org + row * A + gw;
          unsigned int s32 = 0;  // < 2^32: an item holds < 2^32 configurations
          auto term = [&](int dr, int de, int pw) {
            if (e_ok((int)e - de)) s32 += hh[pw - dr * A - de_words(de)];
          };
          if (ok0) {
#pragma unroll
            for (int p = 0; p < (R + 1) * (R + 2) * (R + 3) / 6; ++p)
              s32 += hh[p * S];
          }
          // the planes {a <= b <= c} with n sites of the cluster flipped up
          auto sweep = [&](const int n) {
#pragma unroll
            for (int c = 0; c <= R; ++c)
#pragma unroll
              for (int b = 0; b <= c; ++b)
#pragma unroll
                for (int a = 0; a <= b; ++a) {
                  const int pw =
                      (c * (c + 1) * (c + 2) / 6 + b * (b + 1) / 2 + a) * S;
                  const int fa = R - 2 * a, fb = R - 2 * b, fc = R - 2 * c;
                  if (n == 1) {
                    term(1, fa + I1, pw);
                    term(1, fb + I1, pw);
                    term(1, fc + I1, pw);
                  } else if (n == 2) {
                    term(2, fa + fb + I1, pw);
                    term(2, fa + fc + I1, pw);
                    term(2, fb + fc + I1, pw);
                  } else {
                    term(3, fa + fb + fc, pw);
                  }
                }
          };
          if (ok1) sweep(1);
          if (ok2) sweep(2);
          if (ok3) sweep(3);
          s += s32;
        }
        if (s) atomicAdd(out + m * L.stride() + e, s);
      }
    } else {
      for (unsigned int u = threadIdx.x; u < n_units; u += blockDim.x) {
        const unsigned int mr = u / per_row;
        const unsigned int m = m_lo + mr;
        const unsigned int e = e0 + (u - mr * per_row) * e_step;
        const unsigned int bin = m * L.stride() + e;
        const int row = (int)(m - row_off);  // table row of this bin
        const int gw = (int)isd_bin_word(L, 0u, e);
        unsigned long long s = 0;
        for (unsigned int h = 0; h < L.n_hist(); ++h) {
          const unsigned int* hh = hist + h * L.hist_words();
          if constexpr (PAIR == 0) {
            if (row_ok(row)) s += hh[org + row * A + gw];
          } else {
            const int D0 = L.pair_deg(0);
            const bool ok0 = row_ok(row), ok1 = row_ok(row - 1);
            const int w0 = org + row * A + gw, w1 = w0 - A;
#pragma unroll
            for (int p = 0; p <= D0; ++p) {
              const int plane = p * (int)L.pair_words(0);
              const int f = D0 - 2 * p;
              if (ok0) s += hh[w0 + plane];  // paired site down
              if (ok1 && e_ok((int)e - f))   // ... up: the partner
                s += hh[w1 + plane - de_words(f)];
            }
          }
        }
        if (s) atomicAdd(out + bin, s);
      }
    }
  };

#ifdef ISD_PROBE
  // (probe build) block entry and end of its last flush, ns
  unsigned long long probe_enter, probe_last = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(probe_enter));
#endif
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
      run_body(L, slot_run((t >> 5) * hi_step), 0u);
    }
    __syncthreads();
    flush(L, 0u, L.nbins() / L.stride());
  } else {
    // ---- banded: work items of slots in popcount order ----
    const unsigned int warps = blockDim.x >> 5;
    const unsigned int lane = threadIdx.x & 31;
    const unsigned int base_popc =
        (unsigned int)__popcll(run_begin << L.k());
    __shared__ unsigned int next_slot;  // the item's first unclaimed slot
    __shared__ unsigned int cur_item;
    // Blocks claim items from a zeroed counter (dynamic scheduling), or
    // without one take every gridDim-th item.
    for (unsigned int k = 0;; ++k) {
      if (threadIdx.x == 0) {
        const unsigned int c =
            claim ? atomicAdd(claim, 1u) : blockIdx.x + k * gridDim.x;
        cur_item = c;
        // warp w's first chunk is [w c0, (w + 1) c0) (no claim, no wait);
        // the rest is claimed from next_slot
        if (c < n_items) {
          const unsigned int n = (unsigned int)(items[c].g1 - items[c].g0);
          unsigned int c0 = n / (2u * warps);
          c0 = c0 ? c0 : 1u;
          next_slot = n < warps * c0 ? n : warps * c0;
        }
      }
      zero_hist();
      __syncthreads();
      const unsigned int it = cur_item;
      if (it >= n_items) break;
      const IsdBandItem item = items[it];
      // (calibration launches: SM cycles of this item's walk and flush, for
      // the host to correct its cost model with — capi.cu calibrate_items)
      const long long clk0 = item_clk ? clock64() : 0;
#ifdef ISD_PROBE
      const long long t_item = clock64();
      long long t_first = 0;
#endif
      const unsigned int row_off = base_popc + item.q0;
      // Warps then claim chunks of the item's slots (guided: a chunk is
      // 1/(2W) of what is left, down to one slot), so they finish within
      // about one slot of each other; each chunk starts with an unrank and
      // steps in popcount order.
      const unsigned int n_slots = (unsigned int)(item.g1 - item.g0);
      unsigned int c0 = n_slots / (2u * warps);
      c0 = c0 ? c0 : 1u;
      for (bool first = true;; first = false) {
        unsigned int start = 0, cnt = 0;
        if (first) {
          start = warp * c0;
          cnt = start < n_slots ? min(c0, n_slots - start) : 0u;
          if (cnt == 0) continue;
        } else {
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
        }
        int q = 0;
        unsigned long long v =
            isd_unrank((unsigned int)item.g0 + start, free_bits, &q);
#ifdef ISD_PROBE
        if (t_first == 0) t_first = clock64();
#endif
        // (block-uniform: the item's table in ascending or descending rows)
        if (item.mirror) {
          const IsdMirror<T> M(L);
          for (unsigned int i = 0; i < cnt; ++i) {
            run_body(M, band_run(v), row_off);
            v = isd_next_slot(v, free_bits, &q);
          }
        } else {
          for (unsigned int i = 0; i < cnt; ++i) {
            run_body(L, band_run(v), row_off);
            v = isd_next_slot(v, free_bits, &q);
          }
        }
      }
#ifdef ISD_PROBE
      const long long t_done = clock64();  // this warp's walk ends
#endif
      __syncthreads();
#ifdef ISD_PROBE
      const long long t_walk = clock64();
#endif
      if (item.mirror)
        flush(IsdMirror<T>(L), row_off, L.band_rows());
      else
        flush(L, row_off, L.band_rows());
      __syncthreads();
      if (item_clk && threadIdx.x == 0)
        item_clk[it] = (unsigned long long)(clock64() - clk0);
#ifdef ISD_PROBE
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(probe_last));
      // (probe build) per item: first chunk start, this warp's end, last
      // warp's end, flush end, relative to the item start (SM cycles)
      if (threadIdx.x == 0)
        printf("ISDPROBE blk %u item %u q0 %u slots %u warp %u first %lld "
               "done %lld walk %lld stage1 %lld flush %lld\n", blockIdx.x, it,
               item.q0, (unsigned)(item.g1 - item.g0), warp,
               t_first - t_item, t_done - t_item, t_walk - t_item,
               probe_t1 - t_item, clock64() - t_item);
#endif
    }
  }
#ifdef ISD_PROBE
  // (probe build) block entry and exit on the global nanosecond clock
  {
    unsigned long long probe_exit = probe_last;
    if (!probe_exit) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(probe_exit));
    if (threadIdx.x == 0)
      printf("ISDBLK blk %u enter %llu exit %llu\n", blockIdx.x, probe_enter,
             probe_exit);
  }
#endif
}

#endif  // ISD_K1_BODY_CUH
