// K4 top-k — replaces the lexsort selections of the reference:
//   rerank.build_activation  np.lexsort((arange(n), -scores))[:k1]  (rerank.py:74)
//   rerank.top_neighbors     same key, positives only              (rerank.py:86-87)
//   index.query              np.lexsort((ids, not_self, -final))  (index.py:290-294)
// One CTA per row keeps the running best CAP keys (score desc, tiebreak asc)
// in shared memory: each CAP-sized chunk of the row is filtered against the
// current k-th key, survivors are bitonic-sorted and merged into the best
// list (max(A[i], B[CAP-1-i]) + bitonic merge).  Keys are unique per row, so
// the result equals the reference's stable lexsort prefix.
#include "gift_common.cuh"

namespace gift {

constexpr int TK_THREADS = 256;

template <int CAP>
struct TopkSmem {
  double bs[CAP];
  uint32_t bt[CAP];
  int32_t bj[CAP];
  double cs[CAP];
  uint32_t ct[CAP];
  int32_t cj[CAP];
};

template <int CAP>
__device__ void bitonic_sort_desc(double* s, uint32_t* t, int32_t* j) {
  for (int size = 2; size <= CAP; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < CAP / 2; i += TK_THREADS) {
        int lo = 2 * stride * (i / stride) + (i % stride);
        int hi = lo + stride;
        bool desc = (lo & size) == 0;  // best first in this sub-block
        bool hi_better = key_better(s[hi], t[hi], s[lo], t[lo]);
        if (hi_better == desc) {
          double ts = s[lo]; s[lo] = s[hi]; s[hi] = ts;
          uint32_t tt = t[lo]; t[lo] = t[hi]; t[hi] = tt;
          int32_t tj = j[lo]; j[lo] = j[hi]; j[hi] = tj;
        }
      }
      __syncthreads();
    }
  }
}

template <int CAP>
__device__ void bitonic_merge_desc(double* s, uint32_t* t, int32_t* j) {
  for (int stride = CAP >> 1; stride > 0; stride >>= 1) {
    for (int i = threadIdx.x; i < CAP / 2; i += TK_THREADS) {
      int lo = 2 * stride * (i / stride) + (i % stride);
      int hi = lo + stride;
      if (key_better(s[hi], t[hi], s[lo], t[lo])) {
        double ts = s[lo]; s[lo] = s[hi]; s[hi] = ts;
        uint32_t tt = t[lo]; t[lo] = t[hi]; t[hi] = tt;
        int32_t tj = j[lo]; j[lo] = j[hi]; j[hi] = tj;
      }
    }
    __syncthreads();
  }
}

template <int CAP>
__global__ void __launch_bounds__(TK_THREADS)
    topk_rows_kernel(const double* __restrict__ scores, int64_t n, int k,
                     const int32_t* __restrict__ idrank, const int32_t* __restrict__ self_local,
                     int64_t ord_base, int positive_only, int32_t* __restrict__ out_idx,
                     double* __restrict__ out_val) {
  extern __shared__ __align__(128) char smem_raw[];
  TopkSmem<CAP>& S = *reinterpret_cast<TopkSmem<CAP>*>(smem_raw);
  __shared__ int s_cnt;
  __shared__ double s_ths;
  __shared__ uint32_t s_tht;
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  const double* row = scores + static_cast<int64_t>(b) * n;
  const int64_t self = self_local ? static_cast<int64_t>(self_local[b]) : -1;
  for (int i = tid; i < CAP; i += TK_THREADS) {
    S.bs[i] = -INFINITY;
    S.bt[i] = 0xffffffffu;
    S.bj[i] = -1;
  }
  if (tid == 0) {
    s_ths = -INFINITY;
    s_tht = 0xffffffffu;
    s_cnt = 0;
  }
  __syncthreads();
  for (int64_t c0 = 0; c0 < n; c0 += CAP) {
    const double ths = s_ths;
    const uint32_t tht = s_tht;
    for (int i = tid; i < CAP; i += TK_THREADS) {
      const int64_t jj = c0 + i;
      if (jj < n) {
        const double sc = row[jj];
        const uint32_t tb =
            jj == self ? 0u
                       : 1u + static_cast<uint32_t>(idrank ? static_cast<int64_t>(idrank[jj])
                                                           : ord_base + jj);
        if (key_better(sc, tb, ths, tht)) {
          int pos = atomicAdd(&s_cnt, 1);
          S.cs[pos] = sc;
          S.ct[pos] = tb;
          S.cj[pos] = static_cast<int32_t>(jj);
        }
      }
    }
    __syncthreads();
    const int cnt = s_cnt;
    __syncthreads();  // everyone has read s_cnt before the next chunk appends
    if (cnt > 0) {
      for (int i = cnt + tid; i < CAP; i += TK_THREADS) {
        S.cs[i] = -INFINITY;
        S.ct[i] = 0xffffffffu;
        S.cj[i] = -1;
      }
      __syncthreads();
      bitonic_sort_desc<CAP>(S.cs, S.ct, S.cj);
      // top CAP of (best U cand) = elementwise better of best[i] and
      // cand[CAP-1-i]; staged in registers (two phases, no read/write race)
      double ms[CAP / TK_THREADS > 0 ? CAP / TK_THREADS : 1];
      uint32_t mt[CAP / TK_THREADS > 0 ? CAP / TK_THREADS : 1];
      int32_t mj[CAP / TK_THREADS > 0 ? CAP / TK_THREADS : 1];
#pragma unroll
      for (int q = 0; q < CAP / TK_THREADS; ++q) {
        const int i = tid + q * TK_THREADS;
        const int r = CAP - 1 - i;
        if (key_better(S.cs[r], S.ct[r], S.bs[i], S.bt[i])) {
          ms[q] = S.cs[r]; mt[q] = S.ct[r]; mj[q] = S.cj[r];
        } else {
          ms[q] = S.bs[i]; mt[q] = S.bt[i]; mj[q] = S.bj[i];
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < CAP / TK_THREADS; ++q) {
        const int i = tid + q * TK_THREADS;
        S.bs[i] = ms[q]; S.bt[i] = mt[q]; S.bj[i] = mj[q];
      }
      __syncthreads();
      bitonic_merge_desc<CAP>(S.bs, S.bt, S.bj);
      if (tid == 0) {
        s_ths = S.bs[k - 1];
        s_tht = S.bt[k - 1];
        s_cnt = 0;
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < k; i += TK_THREADS) {
    int32_t j = S.bj[i];
    double v = S.bs[i];
    bool ok = j >= 0 && (!positive_only || v > 0.0);
    out_idx[static_cast<int64_t>(b) * k + i] = ok ? static_cast<int32_t>(ord_base + j) : -1;
    out_val[static_cast<int64_t>(b) * k + i] = ok ? v : 0.0;
  }
}

template <int CAP>
static int launch_topk(const double* scores, int B, int64_t n, int k, const int32_t* idrank,
                       const int32_t* self_local, int64_t ord_base, int positive_only,
                       int32_t* out_idx, double* out_val, cudaStream_t st) {
  const int smem = sizeof(TopkSmem<CAP>);
  GIFT_CUDA_TRY(cudaFuncSetAttribute(topk_rows_kernel<CAP>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  topk_rows_kernel<CAP><<<B, TK_THREADS, smem, st>>>(scores, n, k, idrank, self_local, ord_base,
                                                     positive_only, out_idx, out_val);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

}  // namespace gift

using namespace gift;

extern "C" int gift_topk_rows(const double* scores, int32_t B, int64_t n, int32_t k,
                              const int32_t* idrank, const int32_t* self_local, int64_t ord_base,
                              int32_t positive_only, int32_t* out_idx, double* out_val,
                              void* stream) {
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(k >= 1, GIFT_ERR_INVALID, "k must be >= 1");
  GIFT_REQUIRE(k <= 2048, GIFT_ERR_UNSUPPORTED, "k = %d > 2048", k);
  if (B <= 0) return GIFT_OK;
  if (k <= 256) return launch_topk<256>(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx, out_val, st);
  if (k <= 512) return launch_topk<512>(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx, out_val, st);
  if (k <= 1024) return launch_topk<1024>(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx, out_val, st);
  return launch_topk<2048>(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx, out_val, st);
}
