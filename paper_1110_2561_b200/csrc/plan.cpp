// Host-side lattice validation and kernel-plan compiler.
//
// The lattice arrives as bond classes (include/isingdos_b200.h).  This file
// turns it into the parameter blocks of the two enumeration kernels.  The
// semantic contract is the reference's: m_idx = popcount(index) and e_idx =
// number of unsatisfied bonds (enumeration.py:95-121, 184-204, 232-233).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <vector>
#include <atomic>
#include <functional>
#include <thread>

#include "isd_internal.h"

namespace isd {

static inline int popc64(uint64_t x) { return __builtin_popcountll(x); }


int validate_lattice(const isd_lattice* lat, char* err, size_t errlen) {
  if (!lat) {
    snprintf(err, errlen, "lattice pointer is NULL");
    return ISD_EINVAL;
  }
  const uint32_t n = lat->n_spins;
  if (n < 1 || n > ISD_MAX_SPINS) {
    snprintf(err, errlen, "n_spins=%u outside [1, %d]", n, ISD_MAX_SPINS);
    return ISD_EINVAL;
  }
  if (lat->n_classes < 1 || lat->n_classes > ISD_MAX_CLASSES) {
    snprintf(err, errlen, "n_classes=%u outside [1, %d]", lat->n_classes,
             ISD_MAX_CLASSES);
    return ISD_EINVAL;
  }
  if (lat->reserved != 0) {
    snprintf(err, errlen, "reserved field must be 0");
    return ISD_EINVAL;
  }
  uint32_t bonds = 0;
  for (uint32_t c = 0; c < lat->n_classes; ++c) {
    const isd_bond_class& k = lat->classes[c];
    if (k.shift < 1 || k.shift >= n) {
      snprintf(err, errlen, "class %u: shift %u outside [1, %u)", c, k.shift,
               n);
      return ISD_EINVAL;
    }
    if (k.reserved != 0) {
      snprintf(err, errlen, "class %u: reserved field must be 0", c);
      return ISD_EINVAL;
    }
    // bond (i, i+s) needs i + s < n
    const uint64_t legal = (n - k.shift >= 64) ? ~0ull
                                               : ((1ull << (n - k.shift)) - 1);
    if (k.bond_mask & ~legal) {
      snprintf(err, errlen, "class %u: bond_mask has partners beyond N", c);
      return ISD_EINVAL;
    }
    if (k.jneg_mask & ~k.bond_mask) {
      snprintf(err, errlen, "class %u: jneg_mask not a subset of bond_mask",
               c);
      return ISD_EINVAL;
    }
    bonds += popc64(k.bond_mask);
  }
  if (bonds != lat->n_bonds) {
    snprintf(err, errlen, "n_bonds=%u but the class masks hold %u bonds",
             lat->n_bonds, bonds);
    return ISD_EINVAL;
  }
  if (bonds > 3 * ISD_MAX_SPINS) {
    snprintf(err, errlen, "n_bonds=%u too large", bonds);
    return ISD_EINVAL;
  }
  return ISD_OK;
}

// ---- shared-histogram layout ---------------------------------------------
// The 32 lanes of a warp reduce into one shared histogram at the same time;
// lanes on the same word aggregate in hardware, lanes on different words of
// the same bank serialise (K0 probes 7-10).  The layout and the run bits the
// lanes differ in are picked by replaying a sample of warp instructions and
// minimising the mean over instructions of the largest number of distinct
// words falling into one bank (= shared-memory wavefronts).

static uint64_t rng_next(uint64_t* s) {
  uint64_t x = *s;
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  return *s = x;
}

static uint64_t deposit(uint64_t v, uint64_t mask) {
  uint64_t out = 0;
  for (int b = 0; mask; ++b) {
    const uint64_t low = mask & (~mask + 1);
    if ((v >> b) & 1) out |= low;
    mask ^= low;
  }
  return out;
}

namespace {
struct Bin {
  int m, e, par;
};
}  // namespace

int lane_span(uint64_t lane_mask) {
  return lane_mask ? 64 - __builtin_clzll(lane_mask) : 0;
}

void default_lanes(uint64_t* lane_mask, uint64_t* lane_vec) {
  *lane_mask = 0x1F;
  for (int i = 0; i < 5; ++i) lane_vec[i] = 1ull << i;
}

namespace {
struct Lanes {
  uint64_t mask;    // pivots
  uint64_t vec[5];  // lane bit i flips these run bits (pivot i included)
};
}  // namespace

static Lanes lanes_from_mask(uint64_t mask) {
  Lanes L{mask, {0, 0, 0, 0, 0}};
  uint64_t m = mask;
  for (int i = 0; i < 5; ++i) {
    L.vec[i] = m & (~m + 1);
    m ^= L.vec[i];
  }
  return L;
}

// Adjacency between run bits (run bit b = site b + k).
static std::vector<std::vector<int>> run_neighbors(const isd_lattice* lat,
                                                   int k, int run_bits) {
  std::vector<std::vector<int>> nbr(run_bits);
  for (uint32_t q = 0; q < lat->n_classes; ++q) {
    const isd_bond_class& cl = lat->classes[q];
    for (int i = k; i + (int)cl.shift < (int)lat->n_spins; ++i)
      if ((cl.bond_mask >> i) & 1) {
        const int a = i - k, c = i + (int)cl.shift - k;
        if (a >= run_bits || c >= run_bits) continue;
        nbr[a].push_back(c);
        nbr[c].push_back(a);
      }
  }
  return nbr;
}

// One random move of a plan's lane pattern inside the low `run_bits` run
// bits (the autotuner's GPU hill climb): re-pivot a lane bit (dropping its
// partner), or give it a new random neighbour partner, or none.  Returns
// false when the draw is not a valid pattern.
bool mutate_lanes(const isd_lattice* lat, int run_bits, uint64_t* seed,
                  isd_plan_info* info) {
  const int k = (int)info->k;
  if (run_bits < 6) return false;
  uint64_t pivots = info->lane_mask, partners = 0;
  for (int v = 0; v < 5; ++v) partners |= info->lane_vec[v] & ~pivots;
  const int i = (int)(rng_next(seed) % 5);
  const uint64_t piv_bit = info->lane_vec[i] & pivots;
  if (!piv_bit) return false;
  const int piv = __builtin_ctzll(piv_bit);
  if (rng_next(seed) & 1) {
    const int nb = (int)(rng_next(seed) % run_bits);
    if (((pivots | partners) >> nb) & 1) return false;
    info->lane_mask = (pivots & ~piv_bit) | (1ull << nb);
    info->lane_vec[i] = 1ull << nb;
  } else {
    const std::vector<std::vector<int>> nbr = run_neighbors(lat, k, run_bits);
    std::vector<int> cand;
    for (int c : nbr[piv])
      if (!((pivots >> c) & 1) && !((partners >> c) & 1)) cand.push_back(c);
    const size_t pick = rng_next(seed) % (cand.size() + 1);
    info->lane_vec[i] = piv_bit;
    if (pick < cand.size()) info->lane_vec[i] |= 1ull << cand[pick];
  }
  // the lane vectors must stay a triangular (pivoted) basis: pivots are
  // the lowest bit... any pivot works as long as no vector holds another's
  // pivot
  for (int v = 0; v < 5; ++v)
    if (__builtin_popcountll(info->lane_vec[v] & info->lane_mask) != 1)
      return false;
  return true;
}

// Candidate lane patterns: contiguous windows of 5 run bits, plus (for
// large walks) random 5-subsets — half of them from even-degree sites,
// whose flips keep the lanes' e parity equal — and random "dominoes": each
// lane bit flips its pivot site together with one adjacent run site (lanes
// then differ by pairs of neighbours, which keeps their (m, e) bins closer
// together: fewer distinct words per RED, fewer bank conflicts).
static void lane_candidates(const isd_lattice* lat, const isd_plan_info* info,
                            int run_bits, bool wide, bool single_site,
                            std::vector<Lanes>* out) {
  static const int shifts[] = {0, 3, 6, 9, 12, 15};
  for (int ls : shifts)
    if (run_bits >= ls + 5) out->push_back(lanes_from_mask(0x1Full << ls));
  if (!wide || run_bits < 6) return;
  const int k = (int)info->k;
  std::vector<int> even, all;
  for (int bit = 0; bit < run_bits; ++bit) {
    all.push_back(bit);
    if (!((info->odd_mask >> (bit + k)) & 1)) even.push_back(bit);
  }
  auto seen = [&](uint64_t mask, const uint64_t* vec) {
    for (const Lanes& L : *out)
      if (L.mask == mask && std::equal(L.vec, L.vec + 5, vec)) return true;
    return false;
  };
  uint64_t seed = 0xD1B54A32D192ED03ull;
  for (int pool = 0; pool < 2; ++pool) {
    const std::vector<int>& src = pool == 0 ? even : all;
    if ((int)src.size() < 5) continue;
    for (int r = 0; r < 24; ++r) {
      uint64_t m = 0;
      while (__builtin_popcountll(m) < 5)
        m |= 1ull << src[rng_next(&seed) % src.size()];
      const Lanes L = lanes_from_mask(m);
      if (!seen(L.mask, L.vec)) out->push_back(L);
    }
  }
  if (single_site) return;  // banded tables: lanes flip single sites only
  const std::vector<std::vector<int>> nbr = run_neighbors(lat, k, run_bits);
  for (int r = 0; r < 32; ++r) {
    Lanes L = lanes_from_mask(0);
    uint64_t m = 0;
    while (__builtin_popcountll(m) < 5) m |= 1ull << (rng_next(&seed) % run_bits);
    L = lanes_from_mask(m);
    for (int i = 0; i < 5; ++i) {
      const int p = __builtin_ctzll(L.vec[i]);
      std::vector<int> cand;
      for (int q : nbr[p])
        if (!((m >> q) & 1)) cand.push_back(q);
      if (!cand.empty()) L.vec[i] |= 1ull << cand[rng_next(&seed) % cand.size()];
    }
    if (!seen(L.mask, L.vec)) out->push_back(L);
  }
}

static int site_degree(const isd_lattice* lat, int site) {
  int d = 0;
  for (uint32_t q = 0; q < lat->n_classes; ++q) {
    const isd_bond_class& cl = lat->classes[q];
    d += (int)((cl.bond_mask >> site) & 1);
    if (site >= (int)cl.shift) d += (int)((cl.bond_mask >> (site - cl.shift)) & 1);
  }
  return d;
}

// e change of flipping sites a and b (both down -> both up) beyond the sum
// of the two single flips: each a-b bond is counted by both single flips as
// changing, but flips back: -2 (1 - 2 neg) per bond
static int both_flip_term(const isd_lattice* lat, int a, int b) {
  int t = 0;
  const int lo = a < b ? a : b, hi = a < b ? b : a;
  for (uint32_t q = 0; q < lat->n_classes; ++q) {
    const isd_bond_class& cl = lat->classes[q];
    if (hi - lo == (int)cl.shift && ((cl.bond_mask >> lo) & 1))
      t -= 2 * (1 - 2 * (int)((cl.jneg_mask >> lo) & 1));
  }
  return t;
}

static int energy_of(const isd_lattice* lat, uint64_t x) {
  int e = 0;
  for (uint32_t q = 0; q < lat->n_classes; ++q) {
    const isd_bond_class& cl = lat->classes[q];
    e += popc64(((x ^ (x >> cl.shift)) ^ cl.jneg_mask) & cl.bond_mask);
  }
  return e;
}

// ISD_PAIR: unset = let the model / autotuner choose; 0, 1 or 2 = layouts
// of that pairing mode only (when one fits shared memory)
static int pair_policy() {
  std::string v;
  if (!knob_str("ISD_PAIR", &v) || v.empty()) return -1;
  const int m = std::atoi(v.c_str());
  return m < 0 ? 0 : (m > 3 ? 3 : m);
}

// Index of the multiset {a, b, c} among the multisets of three values in
// 0..R, in (largest, middle, smallest) order: C(hi+2, 3) + C(mid+1, 2) + lo.
static int tri_index(int a, int b, int c) {
  const int lo = std::min(a, std::min(b, c)), hi = std::max(a, std::max(b, c));
  const int mid = a + b + c - lo - hi;
  return hi * (hi + 1) * (hi + 2) / 6 + mid * (mid + 1) / 2 + lo;
}

// Pair mode 3 ("cluster of three"): copy bits 4, 5, 6 are three
// sites that the lattice treats alike — equal degree, each pair of them
// joined by the same number w (0 or 1) of bonds of one sign, and none of
// them adjacent to an unpaired copy site.  One RED then counts the 8
// configurations of the cluster, in the pattern plane of the *multiset* of
// the three sites' unsatisfied external bonds (R = D - 2w external bonds
// each: (R+1)(R+2)(R+3)/6 planes instead of (R+1)^3).  *i1 = the change of
// the cluster's internal unsatisfied bonds when one or two of the three
// sites flip up (2w(1 - 2 neg); 0 when none or all three do).
static bool cluster_of_three(const isd_lattice* lat, const isd_plan_info* info,
                             int* R, int* w, int* i1) {
  const int u = kCopyBits;
  const int s[3] = {info->copy_site[u - 3], info->copy_site[u - 2],
                    info->copy_site[u - 1]};
  auto bonds = [&](int a, int b, int* neg) {
    int cnt = 0;
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    for (uint32_t q = 0; q < lat->n_classes; ++q) {
      const isd_bond_class& cl = lat->classes[q];
      if (hi - lo == (int)cl.shift && ((cl.bond_mask >> lo) & 1)) {
        ++cnt;
        *neg += (int)((cl.jneg_mask >> lo) & 1);
      }
    }
    return cnt;
  };
  int neg01 = 0, neg02 = 0, neg12 = 0;
  const int c01 = bonds(s[0], s[1], &neg01), c02 = bonds(s[0], s[2], &neg02),
            c12 = bonds(s[1], s[2], &neg12);
  if (c01 != c02 || c01 != c12 || c01 > 1) return false;
  if (c01 == 1 && (neg01 != neg02 || neg01 != neg12)) return false;
  const int d0 = site_degree(lat, s[0]);
  if (site_degree(lat, s[1]) != d0 || site_degree(lat, s[2]) != d0) return false;
  for (int t = 0; t < u - 3; ++t)
    for (int i = 0; i < 3; ++i) {
      int ignored = 0;
      if (bonds(info->copy_site[t], s[i], &ignored)) return false;
    }
  const int ext = d0 - 2 * c01;
  for (int i = 0; i < 3; ++i)
    if (info->copy_degree[u - 3 + i] != ext) return false;
  *R = ext;
  *w = c01;
  *i1 = 2 * c01 * (1 - 2 * neg01);
  return true;
}

static void choose_layout(const isd_lattice* lat, isd_plan_info* info,
                          std::vector<isd_plan_info>* ranked, bool wide,
                          int walk_bits, bool climb, int band_rows = 0,
                          int band_span = kBandSpan, bool band_domino = false,
                          uint64_t top = 0, int band_pair = 2) {
  // banded tables: lanes flip single sites (lane m span 5), or with
  // band_domino also a neighbour of the pivot (span 10; rows sized for it)
  const bool single_site = band_rows > 0 && !band_domino;
  // table rows: all N + 1 values of m, or a band of them
  const int n = band_rows ? band_rows - 1 : (int)lat->n_spins;
  const int n_spins = (int)lat->n_spins;
  const int k = (int)info->k;
  const int b = (int)lat->n_bonds;
  const int emax_half = b / 2;  // largest (e - par)/2
  default_lanes(&info->lane_mask, info->lane_vec);
  info->est_wavefronts = 0;
  info->est_per_config = 0;
  info->pair_mode = 0;
  info->band_rows = (uint32_t)band_rows;
  info->band_span = band_rows ? (uint32_t)band_span : 0;
  // paired sites: copy bit 6 (index 0) and, for mode 2, copy bit 5
  const int psite[2] = {info->copy_site[kCopyBits - 1],
                        info->copy_site[kCopyBits - 2]};
  const int pdeg[2] = {site_degree(lat, psite[0]), site_degree(lat, psite[1])};
  const int pboth = both_flip_term(lat, psite[0], psite[1]);
  info->pair_degree[0] = pdeg[0];
  info->pair_degree[1] = pdeg[1];
  info->pair_both = pboth;
  // pair mode 3: copy bits 4-6 as a symmetric cluster (when they are one)
  int tri_r = 0, tri_w = 0, tri_i1 = 0;
  const bool tri_ok = cluster_of_three(lat, info, &tri_r, &tri_w, &tri_i1);
  const int tri_planes = (tri_r + 1) * (tri_r + 2) * (tri_r + 3) / 6;
  // candidate layouts (row_words A, e_words B, plane_words P; paired: plane
  // strides s0 (bit 6) and s1 (bit 5) over the pattern planes)
  struct Cand {
    int a, b, p, span, pair, s0, s1, total;
  };
  static thread_local std::vector<Cand> cand;
  cand.clear();
  if (info->e_mode == 0) {
    for (int t = 0; t < 40; ++t)
      cand.push_back({b + 1 + t, 1, 0, n * (b + 1 + t) + b + 1, 0, 0, 0, 0});
    for (int t = 0; t < 40; ++t)
      cand.push_back({1, n + 1 + t, 0, n + b * (n + 1 + t) + 1, 0, 0, 0, 0});
  } else {
    const bool planes = info->odd_mask != 0;
    for (int t = 0; t < 24; ++t) {
      const int a = emax_half + 1 + t;
      const int span0 = n * a + emax_half + 1;
      for (int q = 0; q < (planes ? 8 : 1); ++q)
        cand.push_back({a, 1, planes ? span0 + 4 * q : 0,
                        planes ? 2 * span0 + 4 * q : span0, 0, 0, 0, 0});
    }
    for (int t = 0; t < 24; ++t) {
      const int bb = n + 1 + t;
      const int span0 = n + emax_half * bb + 1;
      for (int q = 0; q < (planes ? 8 : 1); ++q)
        cand.push_back({1, bb, planes ? span0 + 4 * q : 0,
                        planes ? 2 * span0 + 4 * q : span0, 0, 0, 0, 0});
    }
  }
  const int policy = pair_policy();
  {
    const size_t n_base = cand.size();
    for (size_t ci = 0; ci < n_base; ++ci) {
      Cand c = cand[ci];
      cand[ci].total = c.span;
      // (every other plane offset: the pattern planes spread the banks)
      if (c.p && ((2 * c.p - c.span) / 4) % 2) continue;
      // plane strides: odd residues mod 32 put lanes that differ only in
      // the patterns on different banks (mode 2: p0 + (D0 + 1) p1 times an
      // odd residue: distinct banks while (D0 + 1)(D1 + 1) <= 32)
      for (int r : {1, 9}) {
        c.s0 = ((c.span + 31) & ~31) + r;
        c.pair = 1;
        c.s1 = 0;
        c.total = c.span + pdeg[0] * c.s0;
        if (c.total <= (int)kMaxPairWords) cand.push_back(c);
        c.pair = 2;
        const int end0 = c.span + pdeg[0] * c.s0;
        c.s1 = ((end0 + 31) & ~31) + (r * (pdeg[0] + 1)) % 32;
        c.total = end0 + pdeg[1] * c.s1;
        if (c.total <= (int)(band_rows ? kMaxBandWords : kMaxPair2Words))
          cand.push_back(c);
      }
      // mode 3: one stride over the multiset planes
      if (tri_ok)
        for (int r : {1, 3, 5, 9, 11, 13}) {
          c.pair = 3;
          c.s0 = ((c.span + 31) & ~31) + r;
          c.s1 = 0;
          c.total = c.span + (tri_planes - 1) * c.s0;
          if (c.total <= (int)(band_rows ? kMaxBandWords : kMaxPair2Words))
            cand.push_back(c);
        }
    }
    if (band_rows) {  // banded tables: mode 2, or mode 3 (band_pair)
      std::vector<Cand> keep;
      for (const Cand& c : cand)
        if (c.pair == band_pair) keep.push_back(c);
      cand.swap(keep);
      if (cand.empty()) {
        info->est_per_config = 1e30;
        return;
      }
    }
    if (policy >= 0 && !band_rows) {
      std::vector<Cand> keep;
      for (const Cand& c : cand)
        if (c.pair == policy) keep.push_back(c);
      if (!keep.empty()) cand.swap(keep);
    }
  }
  const int nc = (int)cand.size();
  auto apply = [&](isd_plan_info* dst, const Cand& c) {
    dst->row_words = (uint32_t)c.a;
    dst->e_words = (uint32_t)c.b;
    dst->plane_words = (uint32_t)c.p;
    dst->base_words = (uint32_t)c.span;
    dst->hist_words = (uint32_t)c.total;
    dst->pair_mode = (uint32_t)c.pair;
    dst->pair_words[0] = (uint32_t)c.s0;
    dst->pair_words[1] = (uint32_t)c.s1;
    if (c.pair == 3) {
      // mode 3: external degree R, bonds w between two cluster sites, the
      // internal-bond term, and the plane count
      dst->pair_degree[0] = tri_r;
      dst->pair_degree[1] = tri_w;
      dst->pair_both = tri_i1;
      dst->pair_words[1] = (uint32_t)tri_planes;
    } else {
      dst->pair_degree[0] = pdeg[0];
      dst->pair_degree[1] = pdeg[1];
      dst->pair_both = pboth;
    }
  };
  // default: first candidate
  apply(info, cand[0]);
  // run bits a walk of 2^walk_bits configurations actually varies (a shard
  // fixes the top ones): lane patterns must stay inside them to tile it
  const int run_bits = std::min(n_spins, walk_bits) - k;
  if (run_bits < 5) {
    if (ranked) ranked->push_back(*info);
    return;
  }
  std::vector<Lanes> masks;
  lane_candidates(lat, info, run_bits, wide, single_site, &masks);

  // Score one lane mask against every layout on `warps` sampled warp
  // instructions x kCopySample copies; returns its best cost per
  // configuration and, if `emit`, appends every (layout, mask) alternative
  // to `ranked`.
  constexpr int kWarps = 160, kScreenWarps = 40, kCopySample = 8;
  const int kClimbSteps = (int)knob_long("ISD_CLIMB_STEPS", 40);
  const size_t kClimbStarts = (size_t)knob_long("ISD_CLIMB_STARTS", 3);
  const uint64_t pbit[2] = {1ull << psite[0], 1ull << psite[1]};
  const uint64_t tbit[3] = {1ull << info->copy_site[kCopyBits - 3],
                            1ull << info->copy_site[kCopyBits - 2],
                            1ull << info->copy_site[kCopyBits - 1]};
  std::vector<double> cost(nc);
  // banded tables: a work item may hold its rows in descending order
  // (capi.cu band_items, ISD_BAND_MIRROR), chosen per item — in effect per
  // popcount class of the slot — so a banded layout is scored by the
  // cheaper order of every class: per-class sums for both orders
  const bool mirror_ok = band_rows > 0 && knob_long("ISD_BAND_MIRROR", 1) == 1;
  constexpr int kClasses = 40;
  std::vector<double> cost_f, cost_m;
  if (mirror_ok) {
    cost_f.assign((size_t)nc * kClasses, 0.0);
    cost_m.assign((size_t)nc * kClasses, 0.0);
  }
  // candidates scored by evaluate (the hill climb narrows this to the
  // start pattern's best layouts)
  std::vector<char> active(nc, 1);
  double best = 1e30;
  isd_plan_info best_alt_ = *info;
  auto evaluate = [&](const Lanes& LN, int warps, bool emit) {
    std::fill(cost.begin(), cost.end(), 0.0);
    std::fill(cost_f.begin(), cost_f.end(), 0.0);
    std::fill(cost_m.begin(), cost_m.end(), 0.0);
    const uint64_t lane_mask = LN.mask;
    // the same random stream for every candidate (common random numbers:
    // differences between candidates are then not sampling noise)
    uint64_t seed = 0x9E3779B97F4A7C15ull;
    const uint64_t free_mask = ((1ull << run_bits) - 1) & ~lane_mask;
    uint64_t lane_dep[32];
    for (int lane = 0; lane < 32; ++lane) {
      lane_dep[lane] = 0;
      for (int i = 0; i < 5; ++i)
        if ((lane >> i) & 1) lane_dep[lane] ^= LN.vec[i];
    }
    for (int w = 0; w < warps; ++w) {
      const uint64_t hi = deposit(rng_next(&seed), free_mask);
      const int hq = std::min(popc64(hi), kClasses - 1);
      const uint64_t jb = deposit(rng_next(&seed), info->loop_mask);
      for (int cs = 0; cs < kCopySample; ++cs) {
        uint64_t cbits = 0;
        const uint64_t c = rng_next(&seed) % kCopies;
        for (int t = 0; t < kCopyBits; ++t)
          if ((c >> t) & 1) cbits |= 1ull << info->copy_site[t];
        // distinct bins of the warp instruction for each pairing mode:
        // unpaired (m, e); mode 1 (m, e, p0) of the configuration with the
        // bit-6 site down; mode 2 (m, e, p0, p1) with both sites down; mode
        // 3 (m, e, multiset plane) with the three cluster sites down
        Bin bins[4][32];
        int pat[4][32];
        int nb[4] = {0, 0, 0, 0};
        for (int lane = 0; lane < 32; ++lane) {
          const uint64_t r = hi ^ lane_dep[lane];
          const uint64_t x = (r << k) | jb | cbits | top;
          for (int mode = 0; mode < (tri_ok ? 4 : 3); ++mode) {
            const uint64_t xs =
                mode == 0   ? x
                : mode == 1 ? x & ~pbit[0]
                : mode == 2 ? x & ~(pbit[0] | pbit[1])
                            : x & ~(tbit[0] | tbit[1] | tbit[2]);
            const int e = energy_of(lat, xs);
            int pt = 0;
            if (mode == 1 || mode == 2)
              pt = (pdeg[0] - (energy_of(lat, xs | pbit[0]) - e)) / 2;
            if (mode == 2)
              pt += 64 * ((pdeg[1] - (energy_of(lat, xs | pbit[1]) - e)) / 2);
            if (mode == 3) {
              int nn[3];
              for (int i = 0; i < 3; ++i)
                nn[i] = (tri_r + tri_i1 -
                         (energy_of(lat, xs | tbit[i]) - e)) / 2;
              pt = tri_index(nn[0], nn[1], nn[2]);
            }
            const Bin bn{popc64(xs), e, e & 1};
            bool seen = false;
            for (int t = 0; t < nb[mode] && !seen; ++t)
              seen = bins[mode][t].m == bn.m && bins[mode][t].e == bn.e &&
                     pat[mode][t] == pt;
            if (!seen) {
              pat[mode][nb[mode]] = pt;
              bins[mode][nb[mode]++] = bn;
            }
          }
        }
        for (int ci = 0; ci < nc; ++ci) {
          if (!active[ci]) continue;
          const Cand& cd = cand[ci];
          const Bin* bb = bins[cd.pair];
          const int* pp = pat[cd.pair];
          const int cnt = nb[cd.pair];
          int bank[32] = {0}, bank_m[32] = {0};
          int mx = 0, mx_m = 0;
          for (int t = 0; t < cnt; ++t) {
            int wd;  // the word without its row term
            if (info->e_mode == 0)
              wd = bb[t].e * cd.b;
            else
              wd = ((bb[t].e - bb[t].par) >> 1) * cd.b + bb[t].par * cd.p;
            if (cd.pair == 3)
              wd += pp[t] * cd.s0;
            else
              wd += (pp[t] & 63) * cd.s0 + (pp[t] >> 6) * cd.s1;
            const int v = ++bank[(wd + bb[t].m * cd.a) & 31];
            if (v > mx) mx = v;
            if (mirror_ok) {
              const int vm = ++bank_m[(wd - bb[t].m * cd.a) & 31];
              if (vm > mx_m) mx_m = vm;
            }
          }
          cost[ci] += mx;
          if (mirror_ok) {
            cost_f[(size_t)ci * kClasses + hq] += mx;
            cost_m[(size_t)ci * kClasses + hq] += mx_m;
          }
        }
      }
    }
    double mask_best = 1e30;
    for (int ci = 0; ci < nc; ++ci) {
      if (!active[ci]) continue;
      if (mirror_ok) {  // every class in its cheaper order
        double sum = 0;
        for (int q = 0; q < kClasses; ++q)
          sum += std::min(cost_f[(size_t)ci * kClasses + q],
                          cost_m[(size_t)ci * kClasses + q]);
        cost[ci] = sum;
      }
      const double per_red = cost[ci] / (warps * kCopySample);
      const double per_cfg = per_red / (double)(1 << cand[ci].pair);
      mask_best = std::min(mask_best, per_cfg);
      if (!emit) continue;
      isd_plan_info alt = *info;
      apply(&alt, cand[ci]);
      alt.lane_mask = lane_mask;
      for (int i = 0; i < 5; ++i) alt.lane_vec[i] = LN.vec[i];
      alt.est_wavefronts = per_red;
      alt.est_per_config = per_cfg;
      if (ranked) ranked->push_back(alt);
      if (per_cfg < best - 1e-9) {
        best = per_cfg;
        best_alt_ = alt;
      }
    }
    return mask_best;
  };
  // screen every mask on a quarter of the sample, then score the best 8
  // in full
  if (masks.size() > 8) {
    // (on every third layout: ranks the lane patterns, not the layouts)
    if (nc > 96)
      for (int ci = 0; ci < nc; ++ci) active[ci] = ci % 3 == 0;
    std::vector<std::pair<double, size_t>> screen;
    for (size_t i = 0; i < masks.size(); ++i)
      screen.push_back({evaluate(masks[i], kScreenWarps, false), i});
    std::fill(active.begin(), active.end(), 1);
    std::sort(screen.begin(), screen.end());
    std::vector<Lanes> keep;
    for (size_t i = 0; i < screen.size() && i < 8; ++i)
      keep.push_back(masks[screen[i].second]);
    masks.swap(keep);
  }
  // large walks: hill-climb the best three patterns (re-pivot a lane bit,
  // or give / move / drop its domino partner), scored on the screen sample
  if (climb && wide && run_bits >= 8) {
    const std::vector<std::vector<int>> nbr = run_neighbors(lat, k, run_bits);
    uint64_t seed = 0x2545F4914F6CDD1Dull;
    const size_t n_start = std::min<size_t>(kClimbStarts, masks.size());
    for (size_t si = 0; si < n_start; ++si) {
      Lanes cur = masks[si];
      std::fill(active.begin(), active.end(), 1);
      evaluate(cur, kScreenWarps, false);
      {
        std::vector<std::pair<double, int>> order;
        for (int ci = 0; ci < nc; ++ci)
          order.push_back({cost[ci] / (double)(1 << cand[ci].pair), ci});
        std::sort(order.begin(), order.end());
        std::fill(active.begin(), active.end(), 0);
        for (size_t i = 0; i < order.size() && i < 24; ++i)
          active[order[i].second] = 1;
      }
      double cur_cost = evaluate(cur, kScreenWarps, false);
      for (int step = 0; step < kClimbSteps; ++step) {
        Lanes q = cur;
        const int i = (int)(rng_next(&seed) % 5);
        uint64_t partners = 0;
        for (int v = 0; v < 5; ++v) partners |= q.vec[v] & ~q.mask;
        const int piv = __builtin_ctzll(q.vec[i] & q.mask);
        if (single_site || (rng_next(&seed) & 1)) {  // re-pivot (drops the partner)
          const int nb = (int)(rng_next(&seed) % run_bits);
          if (((q.mask | partners) >> nb) & 1) continue;
          q.mask = (q.mask & ~(1ull << piv)) | (1ull << nb);
          q.vec[i] = 1ull << nb;
        } else {  // partner: new random neighbour of the pivot, or none
          std::vector<int> cand;
          for (int c : nbr[piv])
            if (!((q.mask >> c) & 1)) cand.push_back(c);
          const size_t pick = rng_next(&seed) % (cand.size() + 1);
          q.vec[i] = 1ull << piv;
          if (pick < cand.size()) q.vec[i] |= 1ull << cand[pick];
        }
        const double c = evaluate(q, kScreenWarps, false);
        if (c < cur_cost) {
          cur = q;
          cur_cost = c;
        }
      }
      bool dup = false;
      for (const Lanes& m : masks)
        dup = dup || (m.mask == cur.mask && std::equal(m.vec, m.vec + 5, cur.vec));
      if (!dup) masks.push_back(cur);
    }
    std::fill(active.begin(), active.end(), 1);
  }
  for (const Lanes& m : masks) evaluate(m, kWarps, true);
  if (best < 1e29) *info = best_alt_;
}

// Hoisted split: 7 copy sites and l loop sites inside the low k bits, the
// rest per-thread.
int plan_loop_bits(const isd_lattice* lat, uint64_t n_configs_hint) {
  const int n = (int)lat->n_spins;
  const int u = kCopyBits;
  int log_configs = 0;
  while (log_configs < 63 && (1ull << (log_configs + 1)) <= n_configs_hint)
    ++log_configs;
  if (log_configs > n) log_configs = n;
  // >= 2^22 runs of 2^k configurations: ~28 per thread on 148 SMs, so the
  // grid-stride tail costs < 4% (at ~3.5 runs per thread it cost ~13%)
  int l = log_configs - u - 22;
  // tuning / test knob: force the loop width
  l = (int)knob_long("ISD_LOOP_BITS", l);
  if (l > 7) l = 7;
  if (l < 0) l = 0;
  return l;
}

// Copy-site neighbourhoods for a chosen set of 7 copy sites: every bond
// touching a copy site.  Partner also a copy site -> copy/copy bond folded
// into KT; else the partner is counted through n_q (upward or downward).
static void set_copy_sites(const isd_lattice* lat, isd_plan_info* info,
                           const int* sites, uint32_t e_mode) {
  const int n = (int)lat->n_spins;
  const int u = kCopyBits;
  const int k = (int)info->k;
  for (int t = 0; t < u; ++t) {
    info->copy_site[t] = sites[t];
    info->copy_degree[t] = 0;
    info->copy_nbr1[t] = info->copy_jneg1[t] = 0;
    info->copy_nbr2[t] = info->copy_jneg2[t] = 0;
  }
  info->e_mode = e_mode;
  uint64_t copy_mask = 0;
  int slot[64];
  for (int i = 0; i < 64; ++i) slot[i] = -1;
  for (int t = 0; t < u; ++t) {
    copy_mask |= 1ull << sites[t];
    slot[sites[t]] = t;
  }
  info->loop_mask = ((1ull << k) - 1) & ~copy_mask;
  struct CC { int p, q, neg; };
  CC cc[ISD_MAX_CLASSES * kCopyBits];
  int ncc = 0;
  for (uint32_t c = 0; c < lat->n_classes; ++c) {
    const isd_bond_class& cl = lat->classes[c];
    for (int i = 0; i < n; ++i) {
      if (!((cl.bond_mask >> i) & 1)) continue;
      const int j = i + (int)cl.shift;
      const int ng = (int)((cl.jneg_mask >> i) & 1);
      const int ti = slot[i], tj = slot[j];
      if (ti >= 0 && tj >= 0) {
        cc[ncc++] = CC{ti, tj, ng};
        continue;
      }
      for (int side = 0; side < 2; ++side) {
        const int t = side ? tj : ti;
        const int partner = side ? i : j;
        if (t < 0) continue;
        const uint64_t bit = 1ull << partner;
        if (!(info->copy_nbr1[t] & bit)) {
          info->copy_nbr1[t] |= bit;
          if (ng) info->copy_jneg1[t] |= bit;
        } else {
          // a periodic axis of length 2 doubles the bond (lattice.py:105-107)
          info->copy_nbr2[t] |= bit;
          if (ng) info->copy_jneg2[t] |= bit;
        }
        info->copy_degree[t] += 1;
      }
    }
  }
  for (int c = 0; c < kCopies; ++c) {
    int unsat = 0;
    for (int i = 0; i < ncc; ++i)
      unsat += ((c >> cc[i].p) ^ (c >> cc[i].q) ^ cc[i].neg) & 1;
    info->copy_table[c] = __builtin_popcount((unsigned)c) * (int)info->stride +
                          unsat;
  }
}

int compile_plan(const isd_lattice* lat, uint64_t n_configs_hint,
                 isd_plan_info* info, std::vector<isd_plan_info>* ranked,
                 uint64_t top) {
  std::memset(info, 0, sizeof(*info));
  const int n = (int)lat->n_spins;
  const int u = kCopyBits;
  const int l = plan_loop_bits(lat, n_configs_hint);
  const int k = u + l;
  info->u = u;
  info->l = l;
  info->k = k;
  info->stride = lat->n_bonds + 1;
  // The hoisted kernel needs all copy and loop sites inside the low word and
  // at least one run.
  if (n < k + 1 || k > 32) return 1;
  info->run_mask_above_k = (n >= 64 ? ~0ull : ((1ull << n) - 1)) &
                           ~((1ull << k) - 1);

  // site degrees (with multiplicity) and the e parity structure:
  // e_idx = sum_b (s_i ^ s_j ^ neg_b) = sum_i deg_i s_i + #neg  (mod 2)
  int deg[64] = {0};
  int neg = 0;
  for (uint32_t c = 0; c < lat->n_classes; ++c) {
    const isd_bond_class& cl = lat->classes[c];
    for (int i = 0; i < n; ++i)
      if ((cl.bond_mask >> i) & 1) {
        deg[i]++;
        deg[i + cl.shift]++;
      }
    neg += popc64(cl.jneg_mask);
  }
  uint64_t odd = 0;
  for (int i = 0; i < n; ++i)
    if (deg[i] & 1) odd |= 1ull << i;
  info->odd_mask = odd;
  info->e_parity = (uint32_t)(neg & 1);

  // copy sites, three candidate sets (each laid out; the one with fewer
  // predicted wavefronts wins, and the autotuner re-times the best):
  //   even   the first 7 even-degree sites of [0, k) — the e parity is then
  //          constant over a group's copies (e_mode 1);
  //   low    the lowest 7 sites (e_mode 1 only if every site is even);
  //   spread (large walks) greedily mutually non-adjacent sites, even
  //          degree first — fewer copy-copy bonds, different delta mix.
  auto adjacent = [&](int a, int c) {
    for (uint32_t q = 0; q < lat->n_classes; ++q) {
      const isd_bond_class& cl = lat->classes[q];
      const int lo2 = a < c ? a : c, hi2 = a < c ? c : a;
      if (hi2 - lo2 == (int)cl.shift && ((cl.bond_mask >> lo2) & 1)) return true;
    }
    return false;
  };
  // copy-site sets of the low kk bits
  auto build_sets = [&](int kk, std::vector<std::vector<int>>* sets,
                        std::vector<const char*>* names) {
    std::vector<int> even;
    for (int i = 0; i < kk && (int)even.size() < u; ++i)
      if (!((odd >> i) & 1)) even.push_back(i);
    if ((int)even.size() == u) {
      sets->push_back(even);
      names->push_back("even");
    }
    std::vector<int> low;
    for (int t = 0; t < u; ++t) low.push_back(t);
    std::string forced;
    const bool force_low =
        knob_str("ISD_COPY_VARIANT", &forced) && forced == "low";
    if (sets->empty() || low != (*sets)[0] || force_low) {
      sets->push_back(low);
      names->push_back("low");
    }
    if (n_configs_hint >= (1ull << 33)) {
      std::vector<int> spread;
      for (int pass = 0; pass < 3 && (int)spread.size() < u; ++pass)
        for (int i = 0; i < kk && (int)spread.size() < u; ++i) {
          if (std::find(spread.begin(), spread.end(), i) != spread.end())
            continue;
          const bool even_ok = !((odd >> i) & 1) || pass == 2;
          bool free_ok = true;
          for (int j : spread) free_ok = free_ok && !adjacent(i, j);
          if (even_ok && (free_ok || pass == 2)) spread.push_back(i);
        }
      std::sort(spread.begin(), spread.end());
      bool dup = false;
      for (const auto& st : *sets) dup = dup || st == spread;
      if (!dup) {
        sets->push_back(spread);
        names->push_back("spread");
      }
    }
    // the paired slots (6, then 5) take the set's lowest-degree sites:
    // fewer pattern planes
    for (auto& st : *sets)
      std::stable_sort(st.begin(), st.end(),
                       [&](int x, int y) { return deg[x] > deg[y]; });
  };
  // "tri" sets (pair mode 3): copy bits 4-6 = three like sites of the low kk
  // bits (equal degree, pairwise joined alike: a triangle of a periodic
  // axis of length 3, or mutually non-adjacent), copy bits 0-3 = four low
  // sites adjacent to none of them.  Clusters with the fewest external bonds
  // first (fewest pattern planes); two choices of the unpaired sites each
  // (the lowest four; greedily non-adjacent ones).
  auto bond_count = [&](int a, int c, int* negs) {
    int cnt = 0;
    const int lo2 = a < c ? a : c, hi2 = a < c ? c : a;
    for (uint32_t q = 0; q < lat->n_classes; ++q) {
      const isd_bond_class& cl = lat->classes[q];
      if (hi2 - lo2 == (int)cl.shift && ((cl.bond_mask >> lo2) & 1)) {
        ++cnt;
        *negs += (int)((cl.jneg_mask >> lo2) & 1);
      }
    }
    return cnt;
  };
  auto build_tri_sets = [&](int kk, std::vector<std::vector<int>>* sets,
                            std::vector<const char*>* names) {
    struct Tri {
      int s[3], ext;
      std::vector<int> avail;
    };
    std::vector<Tri> tris;
    for (int a = 0; a < kk; ++a)
      for (int c = a + 1; c < kk; ++c)
        for (int h = c + 1; h < kk; ++h) {
          if (deg[a] != deg[c] || deg[a] != deg[h]) continue;
          int n1 = 0, n2 = 0, n3 = 0;
          const int c1 = bond_count(a, c, &n1), c2 = bond_count(a, h, &n2),
                    c3 = bond_count(c, h, &n3);
          if (c1 != c2 || c1 != c3 || c1 > 1) continue;
          if (c1 == 1 && (n1 != n2 || n1 != n3)) continue;
          Tri t{{a, c, h}, deg[a] - 2 * c1, {}};
          for (int i = 0; i < kk; ++i) {
            if (i == a || i == c || i == h) continue;
            if (adjacent(i, a) || adjacent(i, c) || adjacent(i, h)) continue;
            t.avail.push_back(i);
          }
          if ((int)t.avail.size() >= u - 3) tris.push_back(t);
        }
    std::stable_sort(tris.begin(), tris.end(), [](const Tri& x, const Tri& y) {
      return x.ext < y.ext;
    });
    const size_t n_tri = std::min<size_t>(tris.size(), 2);
    for (size_t ti = 0; ti < n_tri; ++ti) {
      const Tri& t = tris[ti];
      std::vector<int> low(t.avail.begin(), t.avail.begin() + (u - 3));
      std::vector<int> spread;
      for (int pass = 0; pass < 2 && (int)spread.size() < u - 3; ++pass)
        for (int i : t.avail) {
          if ((int)spread.size() >= u - 3) break;
          if (std::find(spread.begin(), spread.end(), i) != spread.end())
            continue;
          bool free_ok = true;
          for (int j : spread) free_ok = free_ok && !adjacent(i, j);
          if (free_ok || pass == 1) spread.push_back(i);
        }
      std::sort(spread.begin(), spread.end());
      for (const std::vector<int>* un : {&low, &spread}) {
        std::vector<int> st(*un);
        st.insert(st.end(), t.s, t.s + 3);
        bool dup = false;
        for (const auto& have_set : *sets) dup = dup || have_set == st;
        if (dup) continue;
        sets->push_back(st);
        names->push_back("tri");
      }
    }
  };
  const int policy = pair_policy();
  std::vector<std::vector<int>> sets;
  std::vector<const char*> names;
  build_sets(k, &sets, &names);
  if (policy < 0 || policy == 3) {
    std::vector<std::vector<int>> tsets;
    std::vector<const char*> tnames;
    build_tri_sets(k, &tsets, &tnames);
    if (policy == 3 && !tsets.empty()) {  // forced: cluster sets only
      sets.clear();
      names.clear();
    }
    sets.insert(sets.end(), tsets.begin(), tsets.end());
    names.insert(names.end(), tnames.begin(), tnames.end());
  }
  isd_plan_info best_info;
  bool have = false;
  std::vector<isd_plan_info> all;
  int walk_bits = 0;
  while (walk_bits < 63 && (1ull << (walk_bits + 1)) <= n_configs_hint)
    ++walk_bits;
  // (test knob ISD_PLAN_WIDE=1: plan a small lattice as a large walk, with
  // random and domino lane patterns, so the CPU replay can check them)
  const bool wide = n_configs_hint >= (1ull << 33) ||
                    knob_long("ISD_PLAN_WIDE", 0) == 1;
  // Each (copy-site set, band shape) variant is searched independently, so
  // a batch of them runs on parallel host threads (the layout search of a
  // large walk is seconds of CPU); results merge in submission order, so
  // the plan does not depend on the thread count.
  struct Variant {
    isd_plan_info base;
    std::vector<int> set;
    bool climb;
    int band_rows, band_span;
    bool band_domino;
    int band_pair;
    isd_plan_info out;
    std::vector<isd_plan_info> all;
  };
  std::vector<Variant> batch;
  auto try_variant = [&](const isd_plan_info& base, const std::vector<int>& set,
                         bool climb, int band_rows, int band_span = kBandSpan,
                         bool band_domino = false, int band_pair = 2) {
    batch.push_back({base, set, climb, band_rows, band_span, band_domino,
                     band_pair, base, {}});
  };
  // What a plan is chosen by.  Large walks: modelled wavefronts per
  // configuration.  Small walks are bound by what every block does once —
  // zeroing its table, flushing it, adding its bins to the global table —
  // which grows with the pattern planes: SM cycles of the walk (32 lanes a
  // clock on each of ~148 SMs) plus about one cycle per table word (two
  // resident blocks, ~0.5 cycles per word each; measured on c1/c2: the
  // unpaired table walks 2^25 configurations in 21 us, the 25-plane mode-2
  // table in 31 us, and the modes cross near 2^27.5 configurations).
  auto score = [&](const isd_plan_info& x) {
    if (wide) return x.est_per_config;
    return x.est_per_config * (double)n_configs_hint / (32.0 * 148.0) +
           (double)x.hist_words;
  };
  auto run_batch = [&]() {
    auto one = [&](Variant& v) {
      v.out = v.base;
      bool all_even = true;
      for (int site : v.set) all_even = all_even && !((odd >> site) & 1);
      set_copy_sites(lat, &v.out, v.set.data(), all_even ? 1 : 0);
      choose_layout(lat, &v.out, &v.all, wide, walk_bits, v.climb,
                    v.band_rows, v.band_span, v.band_domino, top,
                    v.band_pair);
    };
    if (batch.size() == 1) {
      one(batch[0]);
    } else {
      std::vector<std::thread> pool;
      for (Variant& v : batch) pool.emplace_back(one, std::ref(v));
      for (std::thread& t : pool) t.join();
    }
    for (Variant& v : batch) {
      all.insert(all.end(), v.all.begin(), v.all.end());
      if (v.out.est_per_config >= 1e29) continue;  // no layout of that kind
      if (!have || score(v.out) < score(best_info) - 1e-9) {
        best_info = v.out;
        have = true;
      }
    }
    batch.clear();
  };
  // (large walks also hill-climb each set's lane patterns; the model's
  // estimates are only good to a few percent, so every set keeps its best
  // climbed candidates in the list the GPU autotuner times)
  // test / tuning knob: ISD_COPY_VARIANT=even|low|spread forces one set
  std::string force_s;
  const char* force =
      knob_str("ISD_COPY_VARIANT", &force_s) && !force_s.empty()
          ? force_s.c_str()
          : nullptr;
  const long band_knob = knob_long("ISD_BAND", -1);  // 0 never, 1 always
  if (band_knob != 1)
    for (size_t v = 0; v < sets.size(); ++v)
      if (!force || std::strcmp(force, names[v]) == 0)
        try_variant(*info, sets[v], wide, 0);
  run_batch();
  // Banded modes 2 and 3: when no unbanded table of that mode fits (c5: 49
  // planes of all 37 rows), a power-of-two walk can still run it with a
  // table of band_rows rows per work item; a shorter loop (l = 5) keeps the
  // band narrow.  Requires an aligned power-of-two range (checked at
  // launch).
  const bool pow2 = n_configs_hint && !(n_configs_hint & (n_configs_hint - 1));
  // Two band shapes: single-site lanes (lane m span 5) with items of up to
  // kBandSpan + 1 popcount classes and l = 5; or domino lanes (span 10)
  // with one class per item and l = 4, so that the 49-plane table of a
  // degree-6 lattice still fits shared memory.  The domino shape is off by
  // default: on c5 the few layouts that fit 20 rows score 1.24 wavefronts
  // per RED against 1.11 for the single-site shape (the model then picks
  // single-site lanes anyway).  ISD_BAND_DOMINO=1 adds it, 2 keeps only it.
  // Banded mode 3 (cluster sets only): the same shapes with one row fewer
  // (u - 3 unpaired copy bits); its multiset planes are few enough that
  // the domino shape keeps the default span and loop width.
  const long domino_knob = knob_long("ISD_BAND_DOMINO", 0);
  for (int bp = 2; bp <= 3; ++bp) {
    // (mode 2 banded only where no unbanded table of that mode fits; mode 3
    // banded always: its short loop walks all its sites in Gray order and
    // its items may mirror their rows — c4 runs 6% faster banded)
    if (!(band_knob != 0 && pow2 && (policy < 0 || policy == bp) &&
          (band_knob == 1 ||
           (wide && (!have || (int)best_info.pair_mode < bp || bp == 3)))))
      continue;
    for (int shape = 0; shape < 2; ++shape) {
      const bool domino = shape == 1;
      if ((domino && domino_knob == 0) || (!domino && domino_knob == 2))
        continue;
      const int span = (domino && bp == 2)
                           ? 0
                           : (int)knob_long("ISD_BAND_SPAN", kBandSpan);
      // (not capped by the grid-stride loop width l: a banded launch deals
      // work items of slots to blocks, so it has no grid-stride tail; on
      // 2^33-configuration shards l = 5 instead of 4 walks 3.5% faster)
      const long lb_knob = knob_long(
          domino ? "ISD_BAND_DOMINO_LOOP_BITS" : "ISD_BAND_LOOP_BITS", -1);
      const int lb =
          lb_knob >= 0 ? (int)lb_knob : ((domino && bp == 2) ? 4 : 5);
      const int kb = u + lb;
      const int rows = span + (domino ? 10 : 5) + lb + (u - bp) + 1;
      if (walk_bits - kb - 5 >= 1 && kb <= 32 && rows <= n + 1) {
        isd_plan_info base = *info;
        base.l = (uint32_t)lb;
        base.k = (uint32_t)kb;
        base.run_mask_above_k = (n >= 64 ? ~0ull : ((1ull << n) - 1)) &
                                ~((1ull << kb) - 1);
        std::vector<std::vector<int>> bsets;
        std::vector<const char*> bnames;
        if (bp == 2)
          build_sets(kb, &bsets, &bnames);
        else
          build_tri_sets(kb, &bsets, &bnames);
        for (size_t v = 0; v < bsets.size(); ++v)
          if (!force || std::strcmp(force, bnames[v]) == 0)
            try_variant(base, bsets[v], wide, rows, span, domino, bp);
      }
    }
    run_batch();
  }
  if (!have) return 1;  // forced variant not available for this lattice
  // (a small walk: every pairing mode of every set competes on the score —
  // within a set the layout search keeps only the fewest wavefronts)
  if (!wide)
    for (const isd_plan_info& x : all)
      if (x.est_per_config < 1e29 && score(x) < score(best_info) - 1e-9)
        best_info = x;
  *info = best_info;
  if (ranked) {
    // best first within each pairing mode, the modes interleaved (the model
    // cannot see occupancy or the issue cost of fewer REDs per loop
    // subset, so the GPU autotuner must time every mode)
    std::stable_sort(all.begin(), all.end(),
                     [](const isd_plan_info& a, const isd_plan_info& b) {
                       return a.est_per_config < b.est_per_config;
                     });
    std::vector<isd_plan_info> by_mode[6], mixed;
    for (const isd_plan_info& x : all)
      if (x.est_per_config < 1e29)
        by_mode[x.band_rows ? (x.pair_mode == 3 ? 5 : 4) : x.pair_mode % 4]
            .push_back(x);
    size_t total = 0;
    for (const auto& g : by_mode) total += g.size();
    for (size_t i = 0; mixed.size() < total; ++i)
      for (int mode : {5, 4, 3, 2, 1, 0})
        if (i < by_mode[mode].size()) mixed.push_back(by_mode[mode][i]);
    if (mixed.size() > 256) mixed.resize(256);
    ranked->assign(mixed.begin(), mixed.end());
  }
  return 0;
}

void fill_canon(const isd_lattice* lat, CanonParams* p) {
  std::memset(p, 0, sizeof(*p));
  p->n_classes = lat->n_classes;
  p->n_spins = lat->n_spins;
  p->stride = lat->n_bonds + 1;
  p->nbins = (lat->n_spins + 1) * p->stride;
  p->hist_words = hist_words_for(p->nbins);
  p->n_hist = (uint32_t)hist_count_for(p->hist_words);
  for (uint32_t c = 0; c < lat->n_classes; ++c) {
    p->shift[c] = lat->classes[c].shift;
    p->mask[c] = lat->classes[c].bond_mask;
    p->jneg[c] = lat->classes[c].jneg_mask;
  }
}

void fill_hoist(const isd_lattice* lat, const isd_plan_info* info,
                HoistParams* p) {
  std::memset(p, 0, sizeof(*p));
  p->k = info->k;
  p->l = info->l;
  p->above_k = info->run_mask_above_k;
  p->loop_mask = (uint32_t)info->loop_mask;
  p->n_classes = lat->n_classes;
  p->stride = info->stride;
  p->nbins = (lat->n_spins + 1) * p->stride;
  p->e_mode = info->e_mode;
  p->e_parity = info->e_parity;
  p->odd_mask = info->e_mode ? info->odd_mask : 0;
  p->row_words = info->row_words;
  p->e_words = info->e_words;
  p->plane_words = info->plane_words;
  p->row_bytes = 4 * info->row_words;
  // e_mode 1: word = m*A + ((e - par)/2)*B + par*P
  //   -> bytes = 4A m + 2B e + par (4P - 2B)
  p->e_bytes = (info->e_mode ? 2 : 4) * info->e_words;
  p->plane_bytes = info->e_mode ? 4 * (int)info->plane_words -
                                      2 * (int)info->e_words
                                : 0;
  p->lane_mask = info->lane_mask;
  for (int i = 0; i < 5; ++i) p->lane_vec[i] = info->lane_vec[i];
  p->hi_step = 1;
  p->hist_words = hist_words_for(info->hist_words);
  p->n_hist = (uint32_t)hist_count_for(p->hist_words);
  const uint64_t loop = info->loop_mask;
  const uint64_t copies = ((1ull << info->k) - 1) & ~loop;
  for (uint32_t c = 0; c < lat->n_classes; ++c) {
    const isd_bond_class& cl = lat->classes[c];
    p->shift[c] = cl.shift;
    p->mask[c] = cl.bond_mask;
    p->jneg[c] = cl.jneg_mask;
    // lower site a loop site, upper site not a copy site
    p->mvar[c] = (uint32_t)(cl.bond_mask & loop & ~(copies >> cl.shift));
  }
  p->has_double = 0;
  for (int q = 0; q < kCopyBits; ++q) {
    p->nm1[q] = info->copy_nbr1[q];
    p->jn1[q] = info->copy_jneg1[q];
    p->nm2[q] = info->copy_nbr2[q];
    p->jn2[q] = info->copy_jneg2[q];
    p->nm1v[q] = (uint32_t)(info->copy_nbr1[q] & loop);
    p->jn1v[q] = (uint32_t)(info->copy_jneg1[q] & loop);
    p->nm2v[q] = (uint32_t)(info->copy_nbr2[q] & loop);
    p->jn2v[q] = (uint32_t)(info->copy_jneg2[q] & loop);
    p->degree[q] = info->copy_degree[q];
    if (info->copy_nbr2[q]) p->has_double = 1;
  }
  // copy_table[c] = popc(c)(B+1) + unsat_cc(c) -> byte offset of copy c
  const int eb = (int)p->e_bytes, rb = (int)p->row_bytes;
  auto unsat_cc = [&](int c) {
    return info->copy_table[c] -
           __builtin_popcount((unsigned)c) * (int)info->stride;
  };
  for (int c = 0; c < kCopies; ++c)
    p->koff[c] = __builtin_popcount((unsigned)c) * rb + eb * unsat_cc(c);
  p->band_rows = info->band_rows;
  p->band_span = info->band_span;
  p->pair = info->pair_mode;
  p->pair_both = info->pair_both;
  for (int i = 0; i < 2; ++i) {
    p->pair_words[i] = info->pair_words[i];
    p->pair_bytes[i] = 4 * info->pair_words[i];
    p->pair_deg[i] = info->pair_degree[i];
  }
  // Gray sites: the lowest min(G, l) loop sites, G = kDefaultGray — mode 3:
  // kMaxGray, its 16 REDs per loop subset leave the walk issue-bound unless
  // nearly every subset is reached by a site flip (c5 1.355 -> 1.163 ms)
  // (ISD_GRAY=0..kMaxGray overrides it)
  {
    long g = knob_long("ISD_GRAY",
                       info->pair_mode == 3 ? kMaxGray : kDefaultGray);
    if (g < 0) g = 0;
    if (g > kMaxGray) g = kMaxGray;
    if (g > (long)info->l) g = (long)info->l;
    p->gray = (uint32_t)g;
    int slot_of[64];
    for (int i = 0; i < 64; ++i) slot_of[i] = -1;
    for (int t = 0; t < kCopyBits; ++t) slot_of[info->copy_site[t]] = t;
    uint64_t rest = loop;
    for (uint32_t gi = 0; gi < p->gray; ++gi) {
      const int j = __builtin_ctzll(rest);
      rest &= rest - 1;
      p->g_bit[gi] = 1u << j;
      p->g_mask |= 1u << j;
      p->g_odd[gi] = info->e_mode ? (int)((info->odd_mask >> j) & 1) : 0;
      for (uint32_t c = 0; c < lat->n_classes; ++c) {
        const isd_bond_class& cl = lat->classes[c];
        for (int side = 0; side < 2; ++side) {
          // bond (i, i + s) with j at either end
          const int i = side ? j - (int)cl.shift : j;
          if (i < 0 || !((cl.bond_mask >> i) & 1)) continue;
          const int partner = side ? i : i + (int)cl.shift;
          const int neg = (int)((cl.jneg_mask >> i) & 1);
          if (slot_of[partner] >= 0) {
            p->g_cdelta[gi][slot_of[partner]] += 1 - 2 * neg;
            p->g_csum[gi] += 1 - 2 * neg;
            continue;
          }
          const uint64_t bit = 1ull << partner;
          if (!(p->g_nm1[gi] & bit)) {
            p->g_nm1[gi] |= bit;
            if (neg) p->g_jn1[gi] |= bit;
          } else {  // a periodic axis of length 2: the doubled bond
            p->g_nm2[gi] |= bit;
            if (neg) p->g_jn2[gi] |= bit;
          }
          p->g_deg[gi] += 1;
        }
      }
      p->g_nm1v[gi] = (uint32_t)(p->g_nm1[gi] & loop);
      p->g_jn1v[gi] = (uint32_t)(p->g_jn1[gi] & loop);
      p->g_nm2v[gi] = (uint32_t)(p->g_nm2[gi] & loop);
      p->g_jn2v[gi] = (uint32_t)(p->g_jn2[gi] & loop);
    }
  }
  // a paired site's RED lands in pattern plane n + u(c): u(c) = its bonds
  // to the copy sites of c left unsatisfied while it is down (the other
  // paired site down too); flipping it changes unsat_cc by (its copy-copy
  // degree) - 2 u(c)
  // (mode 3: the cluster sites touch no unpaired copy site, u(c) = 0)
  for (uint32_t i = 0; i < (info->pair_mode == 3 ? 0u : info->pair_mode); ++i) {
    const int slot = kCopyBits - 1 - (int)i;
    const int bit = 1 << slot;
    const int cc_deg = info->pair_degree[i] - info->copy_degree[slot];
    const int live = 1 << (kCopyBits - (int)info->pair_mode);
    for (int c = 0; c < live; ++c) {
      const int u = (cc_deg - (unsat_cc(c | bit) - unsat_cc(c))) / 2;
      p->koff[c] += (int)p->pair_bytes[i] * u;
    }
  }
}

}  // namespace isd

namespace isd {

// Expected shared-memory wavefronts per RED of a banded mode-2 launch, per
// segment of its slots: the 2^F values of the F non-pivot run bits in
// (popcount, colex) order — the kernel's slot order — cut into n_seg equal
// ranges.  The walk is wavefront-bound (ncu: pipe ~95% busy), so this is
// its cost per slot up to a constant: measured cycles per slot / (1024 x
// this) stayed within ~2% over the c5 walk (ISD_PROBE).  Items cut to equal
// total cost then finish together.  Cost varies with the popcount class
// (how far the lanes' bins spread) and, within a class, with which sites
// are up, hence segments rather than classes.  Fixed seed: the same plan
// gives the same cuts.  Per segment, `samples` warp REDs of a random slot
// in it, loop subset and unpaired copy: the 32 lanes' words (m, e, pattern
// planes) counted per bank.  `cost_mirror` (optional): the same samples with
// the table's rows in descending order (word = -m A + ...), the layout of
// a mirrored work item.
void band_slot_cost(const isd_lattice* lat, const isd_plan_info& info,
                    uint64_t run_begin, uint64_t lane_mask,
                    const uint64_t* lane_vec, int run_bits, int n_seg,
                    int samples, std::vector<double>* cost,
                    std::vector<double>* cost_mirror, const uint8_t* pos) {
  const int k = (int)info.k;
  const uint64_t free_mask =
      ((run_bits >= 64) ? ~0ull : ((1ull << run_bits) - 1)) & ~lane_mask;
  const int F = popc64(free_mask);
  const uint64_t total = 1ull << F;
  if (n_seg < 1) n_seg = 1;
  if ((uint64_t)n_seg > total) n_seg = (int)total;
  cost->assign((size_t)n_seg, 1.0);
  if (cost_mirror) cost_mirror->assign((size_t)n_seg, 1.0);
  // binomials C(n, j), n, j <= F
  std::vector<uint64_t> C((size_t)(F + 1) * (F + 1), 0);
  for (int n = 0; n <= F; ++n)
    for (int j = 0; j <= n; ++j)
      C[(size_t)n * (F + 1) + j] =
          (j == 0 || j == n) ? 1
                             : C[(size_t)(n - 1) * (F + 1) + j - 1] +
                                   C[(size_t)(n - 1) * (F + 1) + j];
  auto binom = [&](int n, int j) -> uint64_t {
    return (j < 0 || j > n) ? 0 : C[(size_t)n * (F + 1) + j];
  };
  auto unrank = [&](uint64_t g) {  // k1_body.cuh isd_unrank
    int q = 0;
    while (q < F && g >= binom(F, q)) g -= binom(F, q++);
    uint64_t v = 0;
    for (int bit = F - 1; bit >= 0 && q > 0; --bit)
      if (g >= binom(bit, q)) {
        v |= 1ull << bit;
        g -= binom(bit, q--);
      }
    return v;
  };
  uint64_t dep[32];
  for (int lane = 0; lane < 32; ++lane) {
    dep[lane] = 0;
    for (int i = 0; i < 5; ++i)
      if ((lane >> i) & 1) dep[lane] ^= lane_vec[i];
  }
  const uint64_t p0bit = 1ull << info.copy_site[kCopyBits - 1];
  const uint64_t p1bit = 1ull << info.copy_site[kCopyBits - 2];
  const int d0 = (int)info.pair_degree[0], d1 = (int)info.pair_degree[1];
  const bool tri = info.pair_mode == 3;
  const uint64_t p2bit = 1ull << info.copy_site[kCopyBits - 3];
  const int unpaired = kCopyBits - (tri ? 3 : 2);
  // segments are independent (each with its own seed): spread them over
  // the host's cores
  auto run_segment = [&](int sg) {
    uint64_t seed = 0x5851F42D4C957F2Dull ^ (0x9E3779B97F4A7C15ull * (sg + 1));
    const uint64_t g0 = total * (uint64_t)sg / (uint64_t)n_seg;
    const uint64_t g1 = total * (uint64_t)(sg + 1) / (uint64_t)n_seg;
    double tot = 0, tot_m = 0;
    for (int s = 0; s < samples; ++s) {
      const uint64_t sv = unrank(g0 + rng_next(&seed) % (g1 - g0));
      uint64_t slot = 0;  // the slot's bits on their run bits
      if (pos) {
        for (int i = 0; i < F; ++i)
          if ((sv >> i) & 1) slot |= 1ull << pos[i];
      } else {
        slot = deposit(sv, free_mask);
      }
      const uint64_t jb = deposit(rng_next(&seed), info.loop_mask);
      uint64_t cb = 0;
      const uint64_t c = rng_next(&seed);
      for (int t = 0; t < unpaired; ++t)
        if ((c >> t) & 1) cb |= 1ull << info.copy_site[t];
      // a lane's word, without its row term, and its row
      int64_t rest[32], row[32];
      for (int lane = 0; lane < 32; ++lane) {
        const uint64_t run = run_begin + (slot ^ dep[lane]);
        const uint64_t x = (run << k) | jb | cb;  // paired sites down
        const int e = energy_of(lat, x);
        const int eh = info.e_mode ? (e - (e & 1)) / 2 : e;
        const int par = info.e_mode ? (e & 1) : 0;
        row[lane] = popc64(x);
        rest[lane] = (int64_t)eh * info.e_words + par * info.plane_words;
        if (tri) {  // d0 = R, pair_both = the internal-bond term
          const int base = d0 + info.pair_both;
          const int n0 = (base - (energy_of(lat, x | p0bit) - e)) / 2;
          const int n1 = (base - (energy_of(lat, x | p1bit) - e)) / 2;
          const int n2 = (base - (energy_of(lat, x | p2bit) - e)) / 2;
          rest[lane] += (int64_t)tri_index(n0, n1, n2) * info.pair_words[0];
        } else {
          const int p0 = (d0 - (energy_of(lat, x | p0bit) - e)) / 2;
          const int p1 = (d1 - (energy_of(lat, x | p1bit) - e)) / 2;
          rest[lane] += (int64_t)p0 * info.pair_words[0] +
                        (int64_t)p1 * info.pair_words[1];
        }
      }
      // wavefronts of the RED: the most distinct words on one bank
      auto wavefronts = [&](int64_t row_words) {
        int64_t words[32];
        for (int lane = 0; lane < 32; ++lane)
          words[lane] = row[lane] * row_words + rest[lane];
        std::sort(words, words + 32);
        int per_bank[32] = {0};
        int worst = 0;
        for (int i = 0; i < 32; ++i)
          if (i == 0 || words[i] != words[i - 1]) {
            const int b = (int)(((words[i] % 32) + 32) % 32);
            worst = std::max(worst, ++per_bank[b]);
          }
        return worst;
      };
      tot += wavefronts((int64_t)info.row_words);
      if (cost_mirror) tot_m += wavefronts(-(int64_t)info.row_words);
    }
    (*cost)[(size_t)sg] = tot / samples;
    if (cost_mirror) (*cost_mirror)[(size_t)sg] = tot_m / samples;
  };
  unsigned nt = std::thread::hardware_concurrency();
  nt = nt < 1 ? 1 : (nt > 32 ? 32 : nt);
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (int sg; (sg = next.fetch_add(1)) < n_seg;) run_segment(sg);
    });
  for (auto& th : pool) th.join();
}

// The slot map of a banded launch as fields of consecutive bits that move
// together (k1_body.cuh IsdSlotMap): free bit i -> run bit pos[i].  Returns
// the number of fields, or -1 if more than 16 would be needed.
int band_slot_fields(const uint8_t* pos, int F, uint32_t* mask, uint32_t* rot) {
  for (int j = 0; j < 16; ++j) mask[j] = rot[j] = 0;
  int n = 0;
  for (int i = 0; i < F;) {
    int j = i;
    while (j + 1 < F && pos[j + 1] == pos[j] + 1) ++j;
    if (n == 16) return -1;
    mask[n] = (uint32_t)(((1ull << (j + 1)) - 1) & ~((1ull << i) - 1));
    rot[n] = (uint32_t)((pos[i] - i) & 31);
    ++n;
    i = j + 1;
  }
  return n;
}

// Order of the free run bits in a banded launch's slots.  Whether an item
// is cheaper with its rows ascending or descending (band_slot_cost) is
// decided by a few run sites — the neighbours of the lane sites — and an
// item is a contiguous range of the (popcount, colex) slot order: with
// those sites on the most significant slot bits the slots of an item agree
// on them, and the per-item choice is nearly a per-slot one (c5: modelled
// wavefronts per RED 1.078 -> ~1.05).  Influence of a free bit = how far
// the mean of (ascending - descending cost) moves with it, over `slots`
// random slots; bits above a quarter of the largest influence go on top,
// strongest last, the rest keep their natural order below.  pos[i] = run
// bit of slot bit i.  Fixed seed: the same plan gives the same order.
void band_slot_order(const isd_lattice* lat, const isd_plan_info& info,
                     uint64_t run_begin, uint64_t lane_mask,
                     const uint64_t* lane_vec, int run_bits, bool reorder,
                     uint8_t* pos) {
  const uint64_t free_mask =
      ((run_bits >= 64) ? ~0ull : ((1ull << run_bits) - 1)) & ~lane_mask;
  const int F = popc64(free_mask);
  std::vector<int> natural;
  for (int b = 0; b < run_bits; ++b)
    if ((free_mask >> b) & 1) natural.push_back(b);
  for (int i = 0; i < F && i < 24; ++i) pos[i] = (uint8_t)natural[(size_t)i];
  if (!reorder || F < 8 || F > 23 || run_bits > 31) return;
  const int k = (int)info.k;
  uint64_t dep[32];
  for (int lane = 0; lane < 32; ++lane) {
    dep[lane] = 0;
    for (int i = 0; i < 5; ++i)
      if ((lane >> i) & 1) dep[lane] ^= lane_vec[i];
  }
  const bool tri = info.pair_mode == 3;
  const uint64_t p0bit = 1ull << info.copy_site[kCopyBits - 1];
  const uint64_t p1bit = 1ull << info.copy_site[kCopyBits - 2];
  const uint64_t p2bit = 1ull << info.copy_site[kCopyBits - 3];
  const int d0 = (int)info.pair_degree[0], d1 = (int)info.pair_degree[1];
  const int unpaired = kCopyBits - (tri ? 3 : 2);
  constexpr int kSlots = 4096, kPer = 6;
  std::vector<double> sum1((size_t)F, 0.0), sum0((size_t)F, 0.0);
  std::vector<int> n1((size_t)F, 0), n0((size_t)F, 0);
  uint64_t seed = 0xD1B54A32D192ED03ull;
  for (int sidx = 0; sidx < kSlots; ++sidx) {
    const uint64_t sv = rng_next(&seed) & ((1ull << F) - 1);
    const uint64_t slot = deposit(sv, free_mask);
    double d = 0;
    for (int rep = 0; rep < kPer; ++rep) {
      const uint64_t jb = deposit(rng_next(&seed), info.loop_mask);
      uint64_t cb = 0;
      const uint64_t c = rng_next(&seed);
      for (int t = 0; t < unpaired; ++t)
        if ((c >> t) & 1) cb |= 1ull << info.copy_site[t];
      int64_t rest[32], row[32];
      for (int lane = 0; lane < 32; ++lane) {
        const uint64_t run = run_begin + (slot ^ dep[lane]);
        const uint64_t x = (run << k) | jb | cb;
        const int e = energy_of(lat, x);
        const int eh = info.e_mode ? (e - (e & 1)) / 2 : e;
        const int par = info.e_mode ? (e & 1) : 0;
        row[lane] = popc64(x);
        rest[lane] = (int64_t)eh * info.e_words + par * info.plane_words;
        if (tri) {
          const int base = d0 + info.pair_both;
          const int a = (base - (energy_of(lat, x | p0bit) - e)) / 2;
          const int b = (base - (energy_of(lat, x | p1bit) - e)) / 2;
          const int cc = (base - (energy_of(lat, x | p2bit) - e)) / 2;
          rest[lane] += (int64_t)tri_index(a, b, cc) * info.pair_words[0];
        } else {
          const int a = (d0 - (energy_of(lat, x | p0bit) - e)) / 2;
          const int b = (d1 - (energy_of(lat, x | p1bit) - e)) / 2;
          rest[lane] += (int64_t)a * info.pair_words[0] +
                        (int64_t)b * info.pair_words[1];
        }
      }
      auto wavefronts = [&](int64_t row_words) {
        int64_t words[32];
        for (int lane = 0; lane < 32; ++lane)
          words[lane] = row[lane] * row_words + rest[lane];
        std::sort(words, words + 32);
        int per_bank[32] = {0};
        int worst = 0;
        for (int i = 0; i < 32; ++i)
          if (i == 0 || words[i] != words[i - 1]) {
            const int b = (int)(((words[i] % 32) + 32) % 32);
            worst = std::max(worst, ++per_bank[b]);
          }
        return worst;
      };
      d += wavefronts((int64_t)info.row_words) -
           wavefronts(-(int64_t)info.row_words);
    }
    for (int i = 0; i < F; ++i)
      if ((sv >> i) & 1) {
        sum1[(size_t)i] += d;
        ++n1[(size_t)i];
      } else {
        sum0[(size_t)i] += d;
        ++n0[(size_t)i];
      }
  }
  std::vector<double> infl((size_t)F, 0.0);
  double top = 0;
  for (int i = 0; i < F; ++i) {
    if (n1[(size_t)i] && n0[(size_t)i])
      infl[(size_t)i] = std::fabs(sum1[(size_t)i] / n1[(size_t)i] -
                                  sum0[(size_t)i] / n0[(size_t)i]);
    top = std::max(top, infl[(size_t)i]);
  }
  if (top <= 0) return;
  std::vector<int> low, high;
  for (int i = 0; i < F; ++i)
    (infl[(size_t)i] > 0.25 * top ? high : low).push_back(i);
  if (high.empty() || low.empty()) return;
  // strongest influence = most significant slot bit; if that breaks the map
  // into too many fields, the influential bits keep their natural order
  for (int attempt = 0; attempt < 2; ++attempt) {
    std::vector<int> hs(high);
    if (attempt == 0)
      std::stable_sort(hs.begin(), hs.end(), [&](int a, int b) {
        return infl[(size_t)a] < infl[(size_t)b];
      });
    uint8_t cand[24];
    int i = 0;
    for (int b : low) cand[i++] = (uint8_t)natural[(size_t)b];
    for (int b : hs) cand[i++] = (uint8_t)natural[(size_t)b];
    uint32_t m[16], r[16];
    if (band_slot_fields(cand, F, m, r) >= 0) {
      for (int j = 0; j < F; ++j) pos[j] = cand[j];
      return;
    }
  }
}

// Work items of a launch over 2^F slots (popcount order): ~n_target items of
// equal cost, cut so that each spans at most span + 1 popcount classes.  The
// slots are cut into w.size() equal segments and a slot of segment j costs
// w[j] (expected wavefronts per RED, band_slot_cost; empty w: equal costs),
// so items where the lanes' bins spread over more banks hold fewer slots.
std::vector<BandItem> band_work_items(int F, int n_target, int span,
                                      const std::vector<double>& w,
                                      double flush_units, bool* exact) {
  *exact = false;
  std::vector<uint64_t> cum(F + 2, 0);  // cum[q] = slots of popcount < q
  uint64_t c = 1;
  for (int q = 0; q <= F; ++q) {
    cum[q + 1] = cum[q] + c;
    c = c * (uint64_t)(F - q) / (uint64_t)(q + 1);
  }
  const uint64_t total = cum[F + 1];
  const uint64_t n_seg = w.empty() ? 1 : (uint64_t)w.size();
  auto seg_lo = [&](uint64_t j) { return total * j / n_seg; };
  auto wseg = [&](uint64_t j) { return w.empty() ? 1.0 : std::max(w[j], 1e-3); };
  // cost of the slots [a, b)
  auto cost = [&](uint64_t a, uint64_t b) {
    double x = 0;
    for (uint64_t j = a * n_seg / total; j < n_seg && seg_lo(j) < b; ++j) {
      const uint64_t lo = std::max(a, seg_lo(j)), hi = std::min(b, seg_lo(j + 1));
      if (hi > lo) x += (double)(hi - lo) * wseg(j);
    }
    return x;
  };
  // cut [g, end) into items: item k gets budget target(k) (the last one
  // runs to `end`), each capped at span + 1 popcount classes
  auto cut = [&](uint64_t g, uint64_t end, int n_items, auto target,
                 std::vector<BandItem>* out) {
    uint64_t j = g * n_seg / total;
    int q = 0;
    double carry = 0;  // overshoot of the previous item (whole slots)
    for (int k = 0; g < end; ++k) {
      while (cum[q + 1] <= g) ++q;
      const uint64_t limit = std::min(end, cum[std::min(F, q + span) + 1]);
      const uint64_t g0 = g;
      double budget = k >= n_items - 1 ? 1e300 : target(k) + carry;
      // (every item takes at least one slot)
      for (bool first = true; g < limit && (first || budget > 0); first = false) {
        while (seg_lo(j + 1) <= g) ++j;
        const double wj = wseg(j);
        const uint64_t room = std::min(limit, seg_lo(j + 1)) - g;
        uint64_t take = budget > 1e200 ? room
                                       : (uint64_t)std::ceil(budget / wj - 1e-9);
        take = std::max<uint64_t>(1, std::min(take, room));
        g += take;
        budget -= (double)take * wj;
      }
      carry = budget < 0 && budget > -1e200 ? budget : 0;
      out->push_back(BandItem{g0, g, (unsigned)q, 0u});
    }
  };
  const double total_w = cost(0, total);
  const double T = total_w / (n_target > 0 ? n_target : 1);
  std::vector<BandItem> plain;
  cut(0, total, 1 << 30, [&](int) { return T; }, &plain);
  // The extreme popcount classes [0, cum[span + 1]) and [cum[F - span],
  // 2^F) hold few slots, and an item may not reach past them: alone they
  // would leave their blocks idle.  They become second items of blocks 0
  // and 1, whose first items are shortened by their cost plus a flush
  // (flush_units: ~20 K SM cycles in slot-walk units, ISD_PROBE), and the
  // rest is cut into exactly n_target items of equal cost (block b walks
  // item b).
  const uint64_t lo_end = cum[std::min(F, span) + 1];
  const uint64_t hi_start = cum[std::max(0, F - span)];
  if (n_target < 3 || hi_start <= lo_end) {
    *exact = (int)plain.size() == n_target;
    return plain;
  }
  const double c_lo = cost(0, lo_end), c_hi = cost(hi_start, total);
  const bool s_lo = c_lo < 0.5 * T, s_hi = c_hi < 0.5 * T;
  if (!s_lo && !s_hi) {
    *exact = (int)plain.size() == n_target;
    return plain;
  }
  const double f = flush_units;
  std::vector<BandItem> smalls;
  std::vector<double> small_cost;
  if (s_lo) {
    smalls.push_back(BandItem{0, lo_end, 0u, 0u});
    small_cost.push_back(c_lo);
  }
  if (s_hi) {
    smalls.push_back(BandItem{hi_start, total, (unsigned)(F - span), 0u});
    small_cost.push_back(c_hi);
  }
  const uint64_t mid_lo = s_lo ? lo_end : 0, mid_hi = s_hi ? hi_start : total;
  double T2 = cost(mid_lo, mid_hi);
  for (double x : small_cost) T2 += x + f;
  T2 /= n_target;
  // (a block's first item must keep at least half its share; otherwise,
  // e.g. on tiny walks where a flush outweighs an item, the plain split)
  for (double x : small_cost)
    if (T2 - x - f < 0.5 * T2) {
      *exact = (int)plain.size() == n_target;
      return plain;
    }
  std::vector<BandItem> items;
  cut(mid_lo, mid_hi, n_target,
      [&](int k) {
        return k < (int)small_cost.size() ? T2 - small_cost[(size_t)k] - f
                                          : T2;
      },
      &items);
  if ((int)items.size() != n_target) {
    *exact = (int)plain.size() == n_target;
    return plain;
  }
  items.insert(items.end(), smalls.begin(), smalls.end());
  *exact = true;
  return items;
}

}  // namespace isd
