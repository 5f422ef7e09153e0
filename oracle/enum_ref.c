/*
 * enum_ref.c — TEST INFRASTRUCTURE ONLY: the C restatement of the
 * reference's exhaustive walk, used as an independent checker and to
 * produce golden tables the reference cannot express (free boundaries,
 * per-bond signs; BASELINE configs 3 and 4).
 *
 * Two formulations, selectable per run:
 *   naive — explicit +/-1 spins, one multiply per bond, E = -sum J_b s_i s_j
 *           (restates /root/reference/pkg/src/isingdos/oracle.py:71-91);
 *   mask  — unsatisfied bonds counted per bond-offset mask with popcount
 *           (restates the bit-word walk of enumeration.py:167-235 on masks).
 * The naive mode validates the mask mode on small lattices; the mask mode
 * walks 2^36 configurations in minutes on the host cores.
 *
 * stdin:  N B mode(0=naive,1=mask) threads start end
 *         then B lines "i j neg" (bit positions of the two sites; neg=1
 *         when the bond's effective coupling is negative)
 * stdout: (N+1)*(B+1) counts, row-major [m_idx][e_idx], one per line.
 */
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXB 128
#define MAXMASK 16

static struct {
  int n, b, mode, nm;
  size_t bins;
  uint64_t start, end;
  int bi[MAXB], bj[MAXB], bn[MAXB];
  unsigned d_of[MAXMASK];
  uint64_t m_of[MAXMASK], j_of[MAXMASK];
  atomic_ullong next;
} G;

#define CHUNK 65536ull

static void* worker(void* arg) {
  uint64_t* h = (uint64_t*)arg;
  for (;;) {
    const uint64_t a = G.start + atomic_fetch_add(&G.next, CHUNK);
    if (a >= G.end) break;
    const uint64_t z = a + CHUNK < G.end ? a + CHUNK : G.end;
    for (uint64_t x = a; x < z; ++x) {
      const int m = __builtin_popcountll(x);
      int e = 0;
      if (G.mode == 1) {
        for (int q = 0; q < G.nm; ++q)
          e += __builtin_popcountll(((x ^ (x >> G.d_of[q])) ^ G.j_of[q]) &
                                    G.m_of[q]);
      } else {
        /* naive: E/|J| = -sum_b sgn_b s_i s_j, e_idx = (E/|J| + B)/2 */
        int sum = 0;
        for (int k = 0; k < G.b; ++k) {
          const int si = ((x >> G.bi[k]) & 1) ? 1 : -1;
          const int sj = ((x >> G.bj[k]) & 1) ? 1 : -1;
          sum += (G.bn[k] ? -1 : 1) * si * sj;
        }
        e = (-sum + G.b) / 2;
      }
      h[(size_t)m * (G.b + 1) + e] += 1;
    }
  }
  return NULL;
}

int main(void) {
  int n, b, mode, threads;
  unsigned long long start, end;
  if (scanf("%d %d %d %d %llu %llu", &n, &b, &mode, &threads, &start, &end) != 6)
    return 2;
  if (n < 1 || n > 40 || b < 0 || b > MAXB) return 2;
  int bi[MAXB], bj[MAXB], bn[MAXB];
  for (int k = 0; k < b; ++k)
    if (scanf("%d %d %d", &bi[k], &bj[k], &bn[k]) != 3) return 2;

  /* mask formulation: bonds grouped by offset d = hi - lo at bit lo */
  int nm = 0;
  unsigned d_of[MAXMASK];
  uint64_t m_of[MAXMASK], j_of[MAXMASK];
  for (int k = 0; k < b; ++k) {
    int lo = bi[k] < bj[k] ? bi[k] : bj[k];
    int hi = bi[k] < bj[k] ? bj[k] : bi[k];
    unsigned d = (unsigned)(hi - lo);
    int placed = 0;
    for (int q = 0; q < nm && !placed; ++q) {
      if (d_of[q] == d && !((m_of[q] >> lo) & 1)) {
        m_of[q] |= 1ull << lo;
        if (bn[k]) j_of[q] |= 1ull << lo;
        placed = 1;
      }
    }
    if (!placed) {
      if (nm == MAXMASK) return 3;
      d_of[nm] = d;
      m_of[nm] = 1ull << lo;
      j_of[nm] = bn[k] ? (1ull << lo) : 0;
      ++nm;
    }
  }

  const size_t bins = (size_t)(n + 1) * (size_t)(b + 1);
  G.n = n; G.b = b; G.mode = mode; G.nm = nm; G.bins = bins;
  G.start = start; G.end = end;
  memcpy(G.bi, bi, sizeof bi); memcpy(G.bj, bj, sizeof bj);
  memcpy(G.bn, bn, sizeof bn);
  memcpy(G.d_of, d_of, sizeof d_of); memcpy(G.m_of, m_of, sizeof m_of);
  memcpy(G.j_of, j_of, sizeof j_of);
  atomic_init(&G.next, 0);
  uint64_t* total = calloc(bins, sizeof(uint64_t));
  if (threads < 1) threads = 1;
  pthread_t th[256];
  uint64_t* part[256];
  if (threads > 256) threads = 256;
  for (int t = 0; t < threads; ++t) {
    part[t] = calloc(bins, sizeof(uint64_t));
    pthread_create(&th[t], NULL, worker, part[t]);
  }
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    for (size_t i = 0; i < bins; ++i) total[i] += part[t][i];
    free(part[t]);
  }
  for (size_t i = 0; i < bins; ++i) printf("%llu\n", (unsigned long long)total[i]);
  free(total);
  return 0;
}
