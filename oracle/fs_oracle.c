/*
 * fs_oracle.c — plain-C restatement of the reference overlap primitives, multi-threaded
 * with OpenMP.  TEST INFRASTRUCTURE ONLY: used by tests/ as an independent checker and by
 * bench.py as the multi-core CPU baseline ("port").  Never linked by the product library.
 *
 * Reference (abbrev. fs/ = /root/reference/pkg/src/floodstream/):
 *   fso_accumulate  <- fs/_kernels_np.py:16-18 looped as fs/analytics.py:118-120
 *   fso_histogram   <- fs/_kernels_np.py:21-23
 *   fso_composite   <- fs/_kernels_np.py:35-47 (float64 grey, floor(x + 0.5))
 *   fso_pair_counts <- fs/_kernels_np.py:26-32
 *   fso_gram        <- the pair_counts loop of fs/analytics.py:174-181, as bit popcounts
 * Build: oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int nthreads(int t) { return t > 0 ? t : omp_get_max_threads(); }

int fso_accumulate(const uint8_t *const *cells, uint32_t k, uint64_t n, uint32_t *counts,
                   int threads) {
#pragma omp parallel for schedule(static) num_threads(nthreads(threads))
  for (int64_t blk = 0; blk < (int64_t)((n + 4095) / 4096); ++blk) {
    uint64_t p0 = (uint64_t)blk * 4096, p1 = p0 + 4096 < n ? p0 + 4096 : n;
    for (uint64_t p = p0; p < p1; ++p) counts[p] = 0;
    for (uint32_t s = 0; s < k; ++s) {
      const uint8_t *c = cells[s];
      for (uint64_t p = p0; p < p1; ++p) counts[p] += c[p] > 0;
    }
  }
  return 0;
}

int fso_histogram(const uint32_t *counts, uint64_t n, uint64_t nbins, int64_t *bins,
                  int threads) {
  memset(bins, 0, nbins * sizeof(int64_t));
  int T = nthreads(threads);
  int64_t *part = (int64_t *)calloc((size_t)T * nbins, sizeof(int64_t));
  if (!part) return 3;
#pragma omp parallel num_threads(T)
  {
    int64_t *mine = part + (size_t)omp_get_thread_num() * nbins;
#pragma omp for schedule(static)
    for (int64_t p = 0; p < (int64_t)n; ++p)
      if (counts[p] < nbins) mine[counts[p]]++;
  }
  for (int t = 0; t < T; ++t)
    for (uint64_t b = 0; b < nbins; ++b) bins[b] += part[(size_t)t * nbins + b];
  free(part);
  return 0;
}

int fso_composite(const uint32_t *counts, uint64_t n, uint64_t n_inputs, uint8_t *rgba,
                  int threads) {
  const double denom = (double)(n_inputs > 0 ? n_inputs : 1);
#pragma omp parallel for schedule(static) num_threads(nthreads(threads))
  for (int64_t p = 0; p < (int64_t)n; ++p) {
    uint32_t c = counts[p];
    uint8_t *o = rgba + (size_t)p * 4;
    if (c == 0) {
      o[0] = o[1] = o[2] = o[3] = 0;
    } else {
      double sat = (double)c / denom;
      double g = floor(255.0 * (1.0 - sat) + 0.5);
      uint8_t gi = (uint8_t)((long long)g & 0xFF);
      o[0] = gi;
      o[1] = gi;
      o[2] = 255;
      o[3] = 255;
    }
  }
  return 0;
}

int fso_pair_counts(const uint8_t *a, const uint8_t *b, uint64_t n, int64_t *inter, int64_t *uni,
                    int threads) {
  int64_t i_ = 0, u_ = 0;
#pragma omp parallel for schedule(static) reduction(+ : i_, u_) num_threads(nthreads(threads))
  for (int64_t p = 0; p < (int64_t)n; ++p) {
    int x = a[p] > 0, y = b[p] > 0;
    i_ += x & y;
    u_ += x | y;
  }
  *inter = i_;
  *uni = u_;
  return 0;
}

/* pack wet bits, then |A_i & A_j| by 64-bit popcounts over all pairs i <= j.
 * Blocked for full-size configs (C2: 256 x 2^26 px, C3: 1024 x 2^24, C4 bands): work
 * units are (block of BM masks) x (block of BM masks) x (segment of words); a unit sums
 * its segment in sub-chunks of CW words (both blocks' chunks stay in L2) and adds the
 * partial counts into the shared Gram atomically.  Same integers as the plain pair loop. */
#define FSO_BM 16
#define FSO_CW 512
int fso_gram(const uint8_t *const *cells, uint32_t k, uint64_t n, int64_t *gram, int threads) {
  const uint64_t words = (n + 63) / 64;
  uint64_t *bits = (uint64_t *)malloc((size_t)k * words * sizeof(uint64_t) + 8);
  if (!bits) return 3;
  int T = nthreads(threads);
  const int64_t wblocks = (int64_t)((words + 4095) / 4096);
#pragma omp parallel for schedule(dynamic, 4) num_threads(T)
  for (int64_t u = 0; u < (int64_t)k * wblocks; ++u) {
    const uint64_t s = (uint64_t)(u / wblocks), w0 = (uint64_t)(u % wblocks) * 4096;
    const uint64_t w1 = w0 + 4096 < words ? w0 + 4096 : words;
    const uint8_t *c = cells[s];
    for (uint64_t w = w0; w < w1; ++w) {
      uint64_t v = 0, p0 = w * 64, p1 = p0 + 64 < n ? p0 + 64 : n;
      for (uint64_t p = p0; p < p1; ++p) v |= (uint64_t)(c[p] > 0) << (p - p0);
      bits[s * words + w] = v;
    }
  }
  memset(gram, 0, (size_t)k * k * sizeof(int64_t));
  const int64_t nb = ((int64_t)k + FSO_BM - 1) / FSO_BM;
  const int64_t bpairs = nb * (nb + 1) / 2;
  /* enough segments that every thread gets several units */
  int64_t segs = (4 * (int64_t)T + bpairs - 1) / bpairs;
  if (segs < 1) segs = 1;
  int64_t seg_words = (int64_t)((words + segs - 1) / segs);
  seg_words = (seg_words + FSO_CW - 1) / FSO_CW * FSO_CW;
  if (seg_words < FSO_CW) seg_words = FSO_CW;
  segs = ((int64_t)words + seg_words - 1) / seg_words;
#pragma omp parallel for schedule(dynamic, 1) num_threads(T)
  for (int64_t u = 0; u < bpairs * segs; ++u) {
    int64_t e = u / segs, sg = u % segs;
    int64_t bi = 0;
    while (e >= nb - bi) { e -= nb - bi; ++bi; }
    const int64_t bj = bi + e;
    const int64_t i0 = bi * FSO_BM, i1 = i0 + FSO_BM < (int64_t)k ? i0 + FSO_BM : (int64_t)k;
    const int64_t j0 = bj * FSO_BM, j1 = j0 + FSO_BM < (int64_t)k ? j0 + FSO_BM : (int64_t)k;
    int64_t acc[FSO_BM][FSO_BM];
    memset(acc, 0, sizeof(acc));
    const uint64_t s0 = (uint64_t)sg * (uint64_t)seg_words;
    const uint64_t s1 = s0 + (uint64_t)seg_words < words ? s0 + (uint64_t)seg_words : words;
    for (uint64_t c0 = s0; c0 < s1; c0 += FSO_CW) {
      const uint64_t c1 = c0 + FSO_CW < s1 ? c0 + FSO_CW : s1;
      for (int64_t i = i0; i < i1; ++i) {
        const uint64_t *x = bits + (size_t)i * words;
        for (int64_t j = (bi == bj ? i : j0); j < j1; ++j) {
          const uint64_t *y = bits + (size_t)j * words;
          int64_t s = 0;
          for (uint64_t w = c0; w < c1; ++w) s += __builtin_popcountll(x[w] & y[w]);
          acc[i - i0][j - j0] += s;
        }
      }
    }
    for (int64_t i = i0; i < i1; ++i)
      for (int64_t j = (bi == bj ? i : j0); j < j1; ++j) {
        const int64_t s = acc[i - i0][j - j0];
        if (!s) continue;
        __atomic_fetch_add(&gram[i * k + j], s, __ATOMIC_RELAXED);
        if (i != j) __atomic_fetch_add(&gram[j * k + i], s, __ATOMIC_RELAXED);
      }
  }
  free(bits);
  return 0;
}
