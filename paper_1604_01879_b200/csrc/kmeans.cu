// Codebook training kernels — the device half of
// shapesearch.codebook.train_codebook (codebook.py:37-108): k-means++ seeding
// and Lloyd iterations in f64.  The host keeps the reference's control flow
// and its numpy RNG stream (codebook.py:48-61 draws); these kernels compute
//   * |x|^2 per row in numpy's pairwise-summation order
//     ((points * points).sum(axis=1), codebook.py:37-45),
//   * per point the nearest center and its squared distance with the
//     reference's formula max(|x|^2 - 2 x.c + |c|^2, 0), ties to the lower
//     center index (argmin, codebook.py:84-85),
//   * the new centers: per cluster the sum of its members in point order
//     (np.add.at, codebook.py:96-98) divided by the member count.
// Only the x.c dot products use a different summation order than the BLAS
// call of the reference, so labels can differ only for points equidistant to
// two centers within a few ulps.
#include "gift_common.cuh"

namespace gift {
namespace {

// numpy pairwise_sum over n f64 terms term(i) (block 128, 8 accumulators,
// halving split rounded to a multiple of 8), iterative with an explicit stack.
template <typename Term>
__device__ double np_pairwise(int n, Term term) {
  struct Frame {
    int off, n, state;
    double left;
  };
  Frame st[24];
  int top = 0;
  st[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (top >= 0) {
    Frame& f = st[top];
    if (f.n <= 128) {
      double res;
      if (f.n < 8) {
        res = 0.0;
        for (int i = 0; i < f.n; ++i) res = __dadd_rn(res, term(f.off + i));
      } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = term(f.off + j);
        const int lim = f.n - f.n % 8;
        for (int i = 8; i < lim; i += 8)
#pragma unroll
          for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], term(f.off + i + j));
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (int i = lim; i < f.n; ++i) res = __dadd_rn(res, term(f.off + i));
      }
      ret = res;
      --top;
      continue;
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[top + 1] = {f.off, n2, 0, 0.0};
      ++top;
    } else if (f.state == 1) {
      f.state = 2;
      f.left = ret;
      st[top + 1] = {f.off + n2, f.n - n2, 0, 0.0};
      ++top;
    } else {
      ret = __dadd_rn(f.left, ret);
      --top;
    }
  }
  return ret;
}

__global__ void rows_sqnorm_kernel(const double* __restrict__ X, int64_t n, int d,
                                   double* __restrict__ out) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double* x = X + r * d;
  out[r] = np_pairwise(d, [&](int i) { return __dmul_rn(x[i], x[i]); });
}

// One warp per point: all k centers, f64 dots (lane-strided partial sums,
// xor-shuffle tree), first index on ties.
constexpr int KM_WARPS = 8;
__global__ void __launch_bounds__(KM_WARPS * 32)
    kmeans_assign_kernel(const double* __restrict__ X, int64_t n, int d,
                         const double* __restrict__ C, int k, const double* __restrict__ xn2,
                         const double* __restrict__ cn2, int32_t* __restrict__ label,
                         double* __restrict__ mind2) {
  const int lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * KM_WARPS + (threadIdx.x >> 5);
  if (i >= n) return;
  const double* x = X + i * d;
  double best = INFINITY;
  int bi = 0;
  for (int c = 0; c < k; ++c) {
    const double* y = C + static_cast<int64_t>(c) * d;
    double dot = 0.0;
    for (int j = lane; j < d; j += 32) dot = fma(x[j], y[j], dot);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    // codebook.py:37-45: (|x|^2 - 2 x.c) + |c|^2, clamped at 0
    double d2 = __dadd_rn(__dsub_rn(xn2[i], __dmul_rn(2.0, dot)), cn2[c]);
    d2 = d2 < 0.0 ? 0.0 : d2;
    if (d2 < best) {
      best = d2;
      bi = c;
    }
  }
  if (lane == 0) {
    if (label) label[i] = bi;
    if (mind2) mind2[i] = best;
  }
}

// Thread per (cluster, dimension): the members' values added in point order
// from 0.0, then divided by the member count.
__global__ void kmeans_update_kernel(const double* __restrict__ X, int d,
                                     const int64_t* __restrict__ order,
                                     const int64_t* __restrict__ off, int k,
                                     double* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(k) * d) return;
  const int c = static_cast<int>(t / d), j = static_cast<int>(t - static_cast<int64_t>(c) * d);
  double s = 0.0;
  for (int64_t m = off[c]; m < off[c + 1]; ++m) s = __dadd_rn(s, X[order[m] * d + j]);
  out[t] = __ddiv_rn(s, static_cast<double>(off[c + 1] - off[c]));
}

}  // namespace
}  // namespace gift

using namespace gift;

extern "C" int gift_rows_sqnorm_f64(const double* X, int64_t n, int32_t d, double* out,
                                    void* stream) {
  GIFT_REQUIRE(n >= 0 && d >= 1, GIFT_ERR_INVALID, "bad shape");
  if (n == 0) return GIFT_OK;
  rows_sqnorm_kernel<<<static_cast<unsigned>(cdiv(n, 128)), 128, 0, as_stream(stream)>>>(X, n, d,
                                                                                       out);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_kmeans_assign(const double* X, int64_t n, int32_t d, const double* C,
                                  int32_t k, const double* xn2, const double* cn2,
                                  int32_t* out_label, double* out_mind2, void* stream) {
  GIFT_REQUIRE(n >= 0 && d >= 1 && k >= 1, GIFT_ERR_INVALID, "bad shape");
  if (n == 0) return GIFT_OK;
  kmeans_assign_kernel<<<static_cast<unsigned>(cdiv(n, KM_WARPS)), KM_WARPS * 32, 0,
                         as_stream(stream)>>>(X, n, d, C, k, xn2, cn2, out_label, out_mind2);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_kmeans_update(const double* X, int64_t n, int32_t d, const int64_t* order,
                                  const int64_t* off, int32_t k, double* out_centers,
                                  void* stream) {
  GIFT_REQUIRE(n >= 1 && d >= 1 && k >= 1, GIFT_ERR_INVALID, "bad shape");
  const int64_t t = static_cast<int64_t>(k) * d;
  kmeans_update_kernel<<<static_cast<unsigned>(cdiv(t, 256)), 256, 0, as_stream(stream)>>>(
      X, d, order, off, k, out_centers);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}
