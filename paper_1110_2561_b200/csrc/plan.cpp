// Host-side lattice validation and kernel-plan compiler.
//
// The lattice arrives as bond classes (include/isingdos_b200.h).  This file
// turns it into the parameter blocks of the two enumeration kernels.  The
// semantic contract is the reference's: m_idx = popcount(index) and e_idx =
// number of unsatisfied bonds (enumeration.py:95-121, 184-204, 232-233).
#include <cstdio>
#include <cstdlib>
#include <cstring>

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
// the same bank serialise.  The kernel addresses word(m, e) = m*S + e' with
// e' = e (or (e - parity)/2 when e_idx has a fixed parity, which halves the
// footprint and doubles the banks a row touches).  S and the run bits the
// lanes differ in are picked here by replaying a sample of warp
// instructions: minimise the mean over instructions of the largest number
// of distinct words falling into one bank (= wavefronts).

static uint64_t rng_next(uint64_t* s) {
  uint64_t x = *s;
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  return *s = x;
}

static void choose_layout(const isd_lattice* lat, isd_plan_info* info) {
  const int n = (int)lat->n_spins;
  const int k = (int)info->k;
  const int b = (int)lat->n_bonds;
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
  bool even = true;
  for (int i = 0; i < n; ++i) even = even && (deg[i] % 2 == 0);
  info->e_halved = even ? 1 : 0;
  info->e_parity = even ? (uint32_t)(neg & 1) : 0;
  const int min_words = even ? (b - (int)info->e_parity) / 2 + 1 : b + 1;
  info->row_words = (uint32_t)min_words;
  info->e_words = 1;
  info->hist_words = (uint32_t)((n + 1) * min_words);
  info->lane_shift = 0;
  info->est_wavefronts = 0;
  const int run_bits = n - k;
  if (run_bits < 5) return;

  // sample: many warps, a random subset of copies each (copies of one warp
  // are strongly correlated, so breadth over warps matters more)
  // candidate strides: m-major (A = S >= row length, B = 1) and e-major
  // (A = 1, B = R >= N + 1)
  constexpr int kWarps = 64, kCopySample = 16, kHalf = 40, kCand = 2 * kHalf;
  int cand_a[kCand], cand_b[kCand];
  for (int si = 0; si < kHalf; ++si) {
    cand_a[si] = min_words + si;
    cand_b[si] = 1;
    cand_a[kHalf + si] = 1;
    cand_b[kHalf + si] = n + 1 + si;
  }
  static const int shifts[] = {0, 3, 6, 9, 12, 15};
  double best = 1e30;
  int m_s[32], e_s[32];
  for (int ls : shifts) {
    if (run_bits < ls + 5) continue;
    double cost[kCand] = {0};
    uint64_t seed = 0x9E3779B97F4A7C15ull ^ (uint64_t)(ls + 1);
    const uint64_t hi_count = 1ull << (run_bits - 5);
    for (int w = 0; w < kWarps; ++w) {
      const uint64_t hi = rng_next(&seed) % hi_count;
      const uint64_t j = (k > kCopyBits) ? rng_next(&seed) % (1ull << (k - kCopyBits)) : 0;
      for (int cs = 0; cs < kCopySample; ++cs) {
        const int c = (int)(rng_next(&seed) % kCopies);
        for (int lane = 0; lane < 32; ++lane) {
          const uint64_t r = ((hi >> ls) << (ls + 5)) | ((uint64_t)lane << ls) |
                             (hi & ((1ull << ls) - 1));
          const uint64_t x = (r << k) | (j << kCopyBits) | (uint64_t)c;
          int e = 0;
          for (uint32_t q = 0; q < lat->n_classes; ++q) {
            const isd_bond_class& cl = lat->classes[q];
            e += popc64(((x ^ (x >> cl.shift)) ^ cl.jneg_mask) & cl.bond_mask);
          }
          m_s[lane] = popc64(x);
          e_s[lane] = even ? (e - (int)info->e_parity) / 2 : e;
        }
        for (int si = 0; si < kCand; ++si) {
          int words[32];
          int nw = 0;
          for (int lane = 0; lane < 32; ++lane) {
            const int wd = m_s[lane] * cand_a[si] + e_s[lane] * cand_b[si];
            bool seen = false;
            for (int t = 0; t < nw && !seen; ++t) seen = words[t] == wd;
            if (!seen) words[nw++] = wd;
          }
          int bank[32] = {0};
          int mx = 0;
          for (int t = 0; t < nw; ++t) {
            const int v = ++bank[words[t] & 31];
            if (v > mx) mx = v;
          }
          cost[si] += mx;
        }
      }
    }
    for (int si = 0; si < kCand; ++si) {
      const double cst = cost[si] / (kWarps * kCopySample);
      if (cst < best - 1e-9) {
        best = cst;
        info->row_words = (uint32_t)cand_a[si];
        info->e_words = (uint32_t)cand_b[si];
        info->lane_shift = (uint32_t)ls;
      }
    }
  }
  info->est_wavefronts = best;
  info->hist_words = (uint32_t)(n * (int)info->row_words +
                                (min_words - 1) * (int)info->e_words + 1);
}

// Hoisted split: u = 7 copy sites, l loop sites, the rest per-thread.  l is
// chosen so that a full walk still has >= ~2^20 runs to spread over 148 SMs.
int plan_loop_bits(const isd_lattice* lat, uint64_t n_configs_hint) {
  const int n = (int)lat->n_spins;
  const int u = kCopyBits;
  int log_configs = 0;
  while (log_configs < 63 && (1ull << (log_configs + 1)) <= n_configs_hint)
    ++log_configs;
  if (log_configs > n) log_configs = n;
  int l = log_configs - u - 20;
  // tuning / test knob: force the loop width
  if (const char* env = std::getenv("ISD_LOOP_BITS")) l = std::atoi(env);
  if (l > 7) l = 7;
  if (l < 0) l = 0;
  return l;
}

int compile_plan(const isd_lattice* lat, uint64_t n_configs_hint,
                 isd_plan_info* info) {
  std::memset(info, 0, sizeof(*info));
  const int n = (int)lat->n_spins;
  const int u = kCopyBits;
  const int l = plan_loop_bits(lat, n_configs_hint);
  const int k = u + l;
  info->u = u;
  info->l = l;
  info->k = k;
  info->stride = lat->n_bonds + 1;
  info->run_mask_above_k = (n >= 64 ? ~0ull : ((1ull << n) - 1)) &
                           ~((1ull << k) - 1);
  info->var_mask = ((1ull << k) - 1) & ~((1ull << u) - 1);

  // Copy-site neighbourhoods.  A bond (i, i+s) with i < u and i+s >= u is a
  // copy/non-copy bond counted through n_p; with i+s < u it is a copy/copy
  // bond folded into KT.  (Bonds with i >= u never touch a copy site: the
  // upper end is above the lower one.)
  struct CC { int p, q, neg; };
  CC cc[ISD_MAX_CLASSES * kCopyBits];
  int ncc = 0;
  for (int p = 0; p < u && p < n; ++p) {
    for (uint32_t c = 0; c < lat->n_classes; ++c) {
      const isd_bond_class& k2 = lat->classes[c];
      if (!((k2.bond_mask >> p) & 1)) continue;
      const int q = p + (int)k2.shift;
      const int neg = (int)((k2.jneg_mask >> p) & 1);
      if (q >= u) {
        const uint64_t bit = 1ull << q;
        if (!(info->copy_nbr1[p] & bit)) {
          info->copy_nbr1[p] |= bit;
          if (neg) info->copy_jneg1[p] |= bit;
        } else {
          // a periodic axis of length 2 doubles the bond (lattice.py:105-107)
          info->copy_nbr2[p] |= bit;
          if (neg) info->copy_jneg2[p] |= bit;
        }
        info->copy_degree[p] += 1;
      } else {
        cc[ncc++] = CC{p, q, neg};
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
  // The hoisted kernel needs all copy and loop sites inside the low word and
  // at least one run.
  if (n < k + 1 || k > 32) return 1;
  choose_layout(lat, info);
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
  const uint32_t u = info->u, k = info->k;
  p->k = k;
  p->l = info->l;
  p->above_k = info->run_mask_above_k;
  p->n_classes = lat->n_classes;
  p->stride = info->stride;
  p->nbins = (lat->n_spins + 1) * p->stride;
  p->row_words = info->row_words;
  p->row_bytes = 4 * info->row_words;
  p->e_words = info->e_words;
  p->e_halved = info->e_halved;
  p->e_parity = info->e_parity;
  p->e_bytes = (info->e_halved ? 2 : 4) * info->e_words;
  p->lane_shift = info->lane_shift;
  p->hist_words = hist_words_for(info->hist_words);
  p->n_hist = (uint32_t)hist_count_for(p->hist_words);
  const uint32_t var = (uint32_t)info->var_mask;
  for (uint32_t c = 0; c < lat->n_classes; ++c) {
    p->shift[c] = lat->classes[c].shift;
    p->mask[c] = lat->classes[c].bond_mask;
    p->jneg[c] = lat->classes[c].jneg_mask;
    p->mvar[c] = (uint32_t)lat->classes[c].bond_mask & var;
  }
  p->has_double = 0;
  for (uint32_t q = 0; q < u; ++q) {
    p->nm1[q] = info->copy_nbr1[q];
    p->jn1[q] = info->copy_jneg1[q];
    p->nm2[q] = info->copy_nbr2[q];
    p->jn2[q] = info->copy_jneg2[q];
    p->nm1v[q] = (uint32_t)info->copy_nbr1[q] & var;
    p->jn1v[q] = (uint32_t)info->copy_jneg1[q] & var;
    p->nm2v[q] = (uint32_t)info->copy_nbr2[q] & var;
    p->jn2v[q] = (uint32_t)info->copy_jneg2[q] & var;
    p->degree[q] = info->copy_degree[q];
    if (info->copy_nbr2[q]) p->has_double = 1;
  }
  // copy_table[c] = popc(c)(B+1) + unsat_cc(c); split it back into the
  // m and e parts and express the subset-sum steps in bytes
  const int eb = (int)p->e_bytes, rb = (int)p->row_bytes;
  auto unsat = [&](int c) {
    return info->copy_table[c] -
           __builtin_popcount((unsigned)c) * (int)info->stride;
  };
  for (int c = 0; c < kCopies; ++c) {
    if (c == 0) {
      p->ktd[0] = eb * unsat(0);
    } else {
      const int top = 31 - __builtin_clz((unsigned)c);
      p->ktd[c] = rb + eb * (unsat(c) - unsat(c ^ (1 << top)));
    }
  }
}

}  // namespace isd
