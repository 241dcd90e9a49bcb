/*
 * oracle/pairwise.c — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Bit-exact CPU restatement of the squared distance the reference quantizer
 * sorts by (codebook.py:121-124):
 *     diffs = centroids.astype(float64) - x ;  d2 = (diffs * diffs).sum(axis=1)
 * numpy reduces each contiguous row with its pairwise summation: rows of
 * n < 8 are summed left to right from 0.0, rows of 8 <= n <= 128 use eight
 * interleaved accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
 * plus a sequential tail, longer rows split at n2 = n/2 - (n/2 % 8).
 * Must be compiled without FMA contraction (-ffp-contract=off).
 */
#include <stdint.h>

static double leaf(const double* x, const float* c, int64_t off, int64_t n) {
  double t;
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      t = (double)c[off + i] - x[off + i];
      r += t * t;
    }
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) {
    t = (double)c[off + j] - x[off + j];
    r[j] = t * t;
  }
  int64_t i = 8;
  const int64_t lim = n - (n % 8);
  for (; i < lim; i += 8) {
    for (int j = 0; j < 8; ++j) {
      t = (double)c[off + i + j] - x[off + i + j];
      r[j] += t * t;
    }
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) {
    t = (double)c[off + i] - x[off + i];
    res += t * t;
  }
  return res;
}

static double pairwise(const double* x, const float* c, int64_t off, int64_t n) {
  if (n <= 128) return leaf(x, c, off, n);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise(x, c, off, n2) + pairwise(x, c, off + n2, n - n2);
}

/* out[i*m + j] = d2(X[i], C[cand[i*m + j]]); cand == NULL means all K (m = K). */
void gift_oracle_sqdist(const double* X, int64_t n, int64_t d, const float* C, int64_t K,
                        const int64_t* cand, int64_t m, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double* x = X + i * d;
    if (cand == 0) {
      for (int64_t k = 0; k < K; ++k) out[i * K + k] = pairwise(x, C + k * d, 0, d);
    } else {
      for (int64_t j = 0; j < m; ++j) {
        int64_t k = cand[i * m + j];
        out[i * m + j] = pairwise(x, C + k * d, 0, d);
      }
    }
  }
}
