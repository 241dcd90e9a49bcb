// Exact set-to-set matching and the evaluation's rank resolution.
//
// gift_exact_sets replaces matching.exact_hausdorff_distance and
// matching.exact_similarity (matching.py:39-61): for every (query view set b,
// target view set n) pair, the f64 dot matrix of the two sets (the
// reference's `q @ p.T` on f64-widened rows), per query view the best target
// dot, then
//   robust     = mean_v (1 - max_u q_v . p_u)       ("robust" Hausdorff)
//   standard   = max_v  (1 - max_u q_v . p_u)       ("standard" Hausdorff)
//   similarity = mean_v clip(max_u q_v . p_u, 0, 1)  (exact_similarity)
// (1 - x is monotone, so min_u (1 - x_u) = 1 - max_u x_u bit for bit.)  One
// CTA per pair, a warp per query view, f64 FMA over d in lane-strided order.
//
// gift_fif_score_f64 is query_fif (matching.py:136-161) in f64 on CUDA cores:
// for every query view that has a non-zero entry, every posting of its ma
// probed cells, the f64 similarity of the f32 posting and the f32 query
// (cosine: clip(q . p, 0, 1); gaussian: exp(-|q - p|^2 / sigma^2)), the
// per-(view, shape) running max (np.maximum.at from zeros: an atomic max on
// the bits of non-negative doubles), then per shape the view-order f64 sum
// over the views divided by V (`total += view_best; total / V`).  A warp per
// posting, f64 FMA over d.  The opt-in exact-precision path (the tensor-core
// scan's contract is 1e-5 relative; this one is f64 rounding).
//
// gift_eval_ranks replaces the per-query lexsort of evaluate_index /
// exact_baseline_report (index.py:317-357): for each query row of scores and
// each of its relevant shapes j, rank(j) = 1 + #{i != self : key_i < key_j}
// with key = (score desc, id rank asc).  One CTA per query: the relevant keys
// sorted in shared memory, every shape of the row binary-searched into them
// (a histogram of "better than" boundaries), prefix sums give the ranks --
// O(N log R) per query, no sort of the row.
#include "gift_common.cuh"

namespace gift {

constexpr int EX_THREADS = 256;

template <typename TQ, typename TP>
__global__ void __launch_bounds__(EX_THREADS)
    exact_sets_kernel(const TQ* __restrict__ Q, const int32_t* __restrict__ q_cnt, int Vq,
                      const TP* __restrict__ P, const int32_t* __restrict__ p_cnt, int Vp, int d,
                      int N, double* __restrict__ out) {
  __shared__ double s_best[EX_THREADS / 32 * 64];
  const int n = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = q_cnt ? q_cnt[b] : Vq;
  const int np = p_cnt ? p_cnt[n] : Vp;
  const TQ* qb = Q + static_cast<int64_t>(b) * Vq * d;
  const TP* pb = P + static_cast<int64_t>(n) * Vp * d;
  double robust = 0.0, standard = -INFINITY, sim = 0.0;
  // query views in rounds of (warps x 64) so the per-view maxima fit smem
  for (int v0 = 0; v0 < nq; v0 += (EX_THREADS / 32) * 64) {
    const int v1 = min(nq, v0 + (EX_THREADS / 32) * 64);
    for (int v = v0 + warp; v < v1; v += EX_THREADS / 32) {
      double best = -INFINITY;
      for (int u = 0; u < np; ++u) {
        double acc = 0.0;
        for (int k = lane; k < d; k += 32)
          acc = fma(static_cast<double>(qb[static_cast<int64_t>(v) * d + k]),
                    static_cast<double>(pb[static_cast<int64_t>(u) * d + k]), acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        best = fmax(best, acc);
      }
      if (lane == 0) s_best[v - v0] = best;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // view order, sequential f64 sums
      for (int v = v0; v < v1; ++v) {
        const double bst = s_best[v - v0];
        const double m = 1.0 - bst;
        robust += m;
        standard = fmax(standard, m);
        sim += fmin(fmax(bst, 0.0), 1.0);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* o = out + (static_cast<int64_t>(b) * N + n) * 3;
    const double cnt = static_cast<double>(nq);
    o[0] = robust / cnt;
    o[1] = standard;
    o[2] = sim / cnt;
  }
}

constexpr int ER_THREADS = 512;
constexpr int ER_MAX_REL = 4096;

struct RelKey {
  double s;
  uint32_t t;
  int32_t slot;
};

__device__ __forceinline__ bool rk_before(double s1, uint32_t t1, double s2, uint32_t t2) {
  return s1 > s2 || (s1 == s2 && t1 < t2);  // key (score desc, id rank asc)
}

__global__ void __launch_bounds__(ER_THREADS)
    eval_ranks_kernel(const double* __restrict__ scores, int64_t N,
                      const int32_t* __restrict__ idrank, const int32_t* __restrict__ self_local,
                      const int32_t* __restrict__ rel, int R, int32_t* __restrict__ out_rank) {
  extern __shared__ __align__(16) unsigned char er_smem[];
  const int b = blockIdx.x;
  const int rp = 1 << (32 - __clz(max(R, 2) - 1));  // power of two >= R
  RelKey* K = reinterpret_cast<RelKey*>(er_smem);
  int32_t* hist = reinterpret_cast<int32_t*>(K + rp);  // [rp + 1]
  const double* row = scores + static_cast<int64_t>(b) * N;
  const int32_t* rb = rel + static_cast<int64_t>(b) * R;
  const int64_t self = self_local ? self_local[b] : -1;
  for (int s = threadIdx.x; s < rp; s += ER_THREADS) {
    const int j = s < R ? rb[s] : -1;
    K[s] = j >= 0 ? RelKey{row[j], static_cast<uint32_t>(idrank[j]), s}
                  : RelKey{-INFINITY, 0xffffffffu, -1};
  }
  for (int s = threadIdx.x; s <= rp; s += ER_THREADS) hist[s] = 0;
  __syncthreads();
  // bitonic sort of the relevant keys, best first (absent entries last)
  for (int size = 2; size <= rp; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < rp / 2; i += ER_THREADS) {
        const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const RelKey a = K[lo], c = K[hi];
        const bool c_first = rk_before(c.s, c.t, a.s, a.t) ||
                             (!rk_before(a.s, a.t, c.s, c.t) && c.slot >= 0 && a.slot < 0);
        if (c_first == asc) {
          K[lo] = c;
          K[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  int nrel = 0;
  for (int s = 0; s < rp; ++s) nrel += K[s].slot >= 0 ? 1 : 0;  // uniform, short
  // every shape i != self: pos = #relevant keys at or before key_i
  for (int64_t i = threadIdx.x; i < N; i += ER_THREADS) {
    if (i == self) continue;
    const double si = row[i];
    if (si != si) continue;  // NaN: excluded
    const uint32_t ti = static_cast<uint32_t>(idrank[i]);
    int lo = 0, hi = nrel;
    while (lo < hi) {  // first position whose key is after key_i
      const int mid = (lo + hi) >> 1;
      if (rk_before(si, ti, K[mid].s, K[mid].t)) hi = mid; else lo = mid + 1;
    }
    // i ranks before every relevant key at positions >= lo that it precedes
    if (lo < nrel) atomicAdd(&hist[lo], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int s = 0; s < nrel; ++s) {
      run += hist[s];
      out_rank[static_cast<int64_t>(b) * R + K[s].slot] = 1 + run;
    }
  }
  __syncthreads();
  for (int s = threadIdx.x; s < R; s += ER_THREADS)
    if (rb[s] < 0) out_rank[static_cast<int64_t>(b) * R + s] = -1;
}

constexpr int F64_THREADS = 256;

__global__ void __launch_bounds__(F64_THREADS)
    fif_f64_best_kernel(const float* __restrict__ Q, int d, const int32_t* __restrict__ cells,
                        int ma, int K, const int64_t* __restrict__ cell_off,
                        const int32_t* __restrict__ post_ord, const float* __restrict__ feat,
                        int64_t ord_base, int64_t n_local, int mode, double inv_s2,
                        unsigned long long* __restrict__ vb) {
  const int64_t bv = blockIdx.x;
  const float* q = Q + bv * d;
  int any = 0;
  for (int k = threadIdx.x; k < d; k += F64_THREADS) any |= q[k] != 0.0f;
  if (!__syncthreads_or(any)) return;  // an all-zero view contributes 0 (matching.py:152)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* row = vb + bv * n_local;
  for (int a = 0; a < ma; ++a) {
    const int c = cells[bv * ma + a];
    if (c < 0 || c >= K) continue;
    for (int64_t p = cell_off[c] + warp; p < cell_off[c + 1]; p += F64_THREADS / 32) {
      const float* f = feat + p * d;
      double acc = 0.0;
      if (mode == GIFT_SIM_COSINE) {
        for (int k = lane; k < d; k += 32)
          acc = fma(static_cast<double>(q[k]), static_cast<double>(f[k]), acc);
      } else {
        for (int k = lane; k < d; k += 32) {
          const double df = static_cast<double>(q[k]) - static_cast<double>(f[k]);
          acc = fma(df, df, acc);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        const double sim = mode == GIFT_SIM_COSINE ? fmin(fmax(acc, 0.0), 1.0) : exp(-acc * inv_s2);
        atomicMax(row + (post_ord[p] - ord_base),
                  static_cast<unsigned long long>(__double_as_longlong(sim)));
      }
    }
  }
}

__global__ void fif_f64_sum_kernel(const unsigned long long* __restrict__ vb, int B, int V,
                                   int64_t n_local, double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(B) * n_local) return;
  const int64_t b = i / n_local, j = i - b * n_local;
  double t = 0.0;
  for (int v = 0; v < V; ++v)
    t += __longlong_as_double(static_cast<long long>(vb[(b * V + v) * n_local + j]));
  out[i] = t / static_cast<double>(V);
}

}  // namespace gift

using namespace gift;

extern "C" size_t gift_fif_score_f64_ws_bytes(int32_t B, int32_t V, int64_t n_local) {
  if (B <= 0 || V <= 0 || n_local <= 0) return 0;
  return static_cast<size_t>(B) * static_cast<size_t>(V) * static_cast<size_t>(n_local) *
         sizeof(unsigned long long);
}

extern "C" int gift_fif_score_f64(const float* Q, int32_t B, int32_t V, int32_t d,
                                  const int32_t* cells, int32_t ma, int32_t K,
                                  const int64_t* cell_off, const int32_t* post_ord,
                                  const float* feat, int64_t ord_base, int64_t n_local,
                                  int32_t mode, double sigma, void* ws, size_t ws_bytes,
                                  double* out, void* stream) {
  GIFT_REQUIRE(mode == GIFT_SIM_COSINE || mode == GIFT_SIM_GAUSSIAN, GIFT_ERR_INVALID,
               "unknown similarity mode %d", mode);
  GIFT_REQUIRE(mode == GIFT_SIM_COSINE || sigma > 0.0, GIFT_ERR_INVALID, "sigma must be > 0");
  GIFT_REQUIRE(d >= 1 && ma >= 1 && K >= 1, GIFT_ERR_INVALID, "bad f64 F-IF score shape");
  if (B <= 0 || n_local <= 0) return GIFT_OK;
  GIFT_REQUIRE(V >= 1, GIFT_ERR_EMPTY, "view set is empty");
  GIFT_REQUIRE(ws_bytes >= gift_fif_score_f64_ws_bytes(B, V, n_local), GIFT_ERR_CAPACITY,
               "f64 F-IF score workspace too small");
  cudaStream_t st = as_stream(stream);
  auto* vb = static_cast<unsigned long long*>(ws);
  GIFT_CUDA_TRY(cudaMemsetAsync(vb, 0, gift_fif_score_f64_ws_bytes(B, V, n_local), st));
  fif_f64_best_kernel<<<static_cast<unsigned>(static_cast<int64_t>(B) * V), F64_THREADS, 0, st>>>(
      Q, d, cells, ma, K, cell_off, post_ord, feat, ord_base, n_local, mode,
      mode == GIFT_SIM_GAUSSIAN ? 1.0 / (sigma * sigma) : 0.0, vb);
  GIFT_LAUNCH_CHECK();
  const int64_t n = static_cast<int64_t>(B) * n_local;
  fif_f64_sum_kernel<<<static_cast<unsigned>(cdiv(n, 256)), 256, 0, st>>>(vb, B, V, n_local, out);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_exact_sets(const void* Q, int32_t qdtype, const int32_t* q_cnt, int32_t B,
                               int32_t Vq, const void* P, int32_t pdtype, const int32_t* p_cnt,
                               int32_t N, int32_t Vp, int32_t d, double* out, void* stream) {
  GIFT_REQUIRE((qdtype == GIFT_F32 || qdtype == GIFT_F64) &&
                   (pdtype == GIFT_F32 || pdtype == GIFT_F64),
               GIFT_ERR_INVALID, "exact sets: f32 or f64 views");
  GIFT_REQUIRE(d >= 1, GIFT_ERR_DIM, "empty views");
  if (B <= 0 || N <= 0) return GIFT_OK;
  GIFT_REQUIRE(Vq >= 1 && Vp >= 1, GIFT_ERR_EMPTY, "view set is empty");
  cudaStream_t st = as_stream(stream);
  dim3 grid(static_cast<unsigned>(N), static_cast<unsigned>(B));
  if (qdtype == GIFT_F32 && pdtype == GIFT_F32)
    exact_sets_kernel<float, float><<<grid, EX_THREADS, 0, st>>>(
        static_cast<const float*>(Q), q_cnt, Vq, static_cast<const float*>(P), p_cnt, Vp, d, N, out);
  else if (qdtype == GIFT_F64 && pdtype == GIFT_F32)
    exact_sets_kernel<double, float><<<grid, EX_THREADS, 0, st>>>(
        static_cast<const double*>(Q), q_cnt, Vq, static_cast<const float*>(P), p_cnt, Vp, d, N,
        out);
  else if (qdtype == GIFT_F32 && pdtype == GIFT_F64)
    exact_sets_kernel<float, double><<<grid, EX_THREADS, 0, st>>>(
        static_cast<const float*>(Q), q_cnt, Vq, static_cast<const double*>(P), p_cnt, Vp, d, N,
        out);
  else
    exact_sets_kernel<double, double><<<grid, EX_THREADS, 0, st>>>(
        static_cast<const double*>(Q), q_cnt, Vq, static_cast<const double*>(P), p_cnt, Vp, d, N,
        out);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_eval_ranks(const double* scores, int32_t B, int64_t N, const int32_t* idrank,
                               const int32_t* self_local, const int32_t* rel, int32_t R,
                               int32_t* out_rank, void* stream) {
  GIFT_REQUIRE(R >= 1 && R <= ER_MAX_REL, GIFT_ERR_UNSUPPORTED,
               "relevant shapes per query = %d outside [1, %d]", R, ER_MAX_REL);
  GIFT_REQUIRE(idrank != nullptr, GIFT_ERR_INVALID, "eval ranks need the id ranks");
  if (B <= 0) return GIFT_OK;
  int rp = 2;
  while (rp < R) rp <<= 1;
  const size_t smem = static_cast<size_t>(rp) * sizeof(RelKey) + (rp + 1) * sizeof(int32_t);
  cudaStream_t st = as_stream(stream);
  GIFT_CUDA_TRY(cudaFuncSetAttribute(eval_ranks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  eval_ranks_kernel<<<static_cast<unsigned>(B), ER_THREADS, smem, st>>>(scores, N, idrank,
                                                                      self_local, rel, R, out_rank);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}
