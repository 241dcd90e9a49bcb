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

struct TopkIn {
  // dense rows (slice pass)
  const double* scores;
  int64_t n, slice_len;
  const int32_t* idrank;
  const int32_t* self_local;
  int64_t ord_base;
  // explicit candidates (merge pass): m per row, idx already global
  const double* cs;
  const uint32_t* ct;
  const int32_t* ci;
  int64_t m;
  const int32_t* counts;  // optional: valid candidates per row (<= m)
  const int64_t* row_off;  // optional: row b starts at row_off[b] + b * row_pad
  int64_t row_pad;         //   (instead of b * m; m then bounds the counts)
};

__device__ __forceinline__ int64_t list_row(const TopkIn& in, int b) {
  return in.row_off ? in.row_off[b] + static_cast<int64_t>(b) * in.row_pad
                    : static_cast<int64_t>(b) * in.m;
}

struct TopkOut {
  int k, positive_only, final_out, nslices;
  int32_t* out_idx;  // final: [B, k]
  double* out_val;
  double* cs;        // partial: [B, nslices, k]
  uint32_t* ct;
  int32_t* ci;
};

template <int CAP, bool DENSE>
__global__ void __launch_bounds__(TK_THREADS) topk_kernel(const TopkIn in, const TopkOut out) {
  extern __shared__ __align__(128) char smem_raw[];
  TopkSmem<CAP>& S = *reinterpret_cast<TopkSmem<CAP>*>(smem_raw);
  __shared__ int s_cnt;
  __shared__ double s_ths;
  __shared__ uint32_t s_tht;
  const int b = blockIdx.y;
  const int sl = blockIdx.x;
  const int tid = threadIdx.x;
  const int k = out.k;
  int64_t e0, e1;
  if (DENSE) {
    e0 = static_cast<int64_t>(sl) * in.slice_len;
    e1 = min64(in.n, e0 + in.slice_len);
  } else {
    e0 = 0;
    e1 = in.counts ? min64(in.m, static_cast<int64_t>(in.counts[b])) : in.m;
  }
  const double* row = DENSE ? in.scores + static_cast<int64_t>(b) * in.n : nullptr;
  const int64_t self = (DENSE && in.self_local) ? static_cast<int64_t>(in.self_local[b]) : -1;
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
  // Stream the keys in sub-chunks of CAP/2; survivors of the running
  // threshold are appended to the candidate buffer, which is sorted and
  // merged into the best list only when it is half full (or at the end).
  constexpr int SUB = CAP / 2;
  for (int64_t c0 = e0; c0 < e1; c0 += SUB) {
    const double ths = s_ths;
    const uint32_t tht = s_tht;
    for (int i = tid; i < SUB; i += TK_THREADS) {
      const int64_t e = c0 + i;
      if (e < e1) {
        double sc;
        uint32_t tb;
        int32_t jj;
        if (DENSE) {
          sc = row[e];
          tb = e == self ? 0u
                         : 1u + static_cast<uint32_t>(in.idrank ? static_cast<int64_t>(in.idrank[e])
                                                                : in.ord_base + e);
          jj = static_cast<int32_t>(in.ord_base + e);
        } else {
          const int64_t at = list_row(in, b) + e;
          sc = in.cs[at];
          jj = in.ci[at];
          tb = in.ct ? in.ct[at] : static_cast<uint32_t>(jj);
        }
        if (jj >= 0 && key_better(sc, tb, ths, tht)) {
          int pos = atomicAdd(&s_cnt, 1);
          S.cs[pos] = sc;
          S.ct[pos] = tb;
          S.cj[pos] = jj;
        }
      }
    }
    __syncthreads();
    const int cnt = s_cnt;
    const bool last = c0 + SUB >= e1;
    __syncthreads();  // everyone has read s_cnt before the next sub-chunk appends
    if (cnt >= SUB || (last && cnt > 0)) {
      for (int i = cnt + tid; i < CAP; i += TK_THREADS) {
        S.cs[i] = -INFINITY;
        S.ct[i] = 0xffffffffu;
        S.cj[i] = -1;
      }
      __syncthreads();
      bitonic_sort_desc<CAP>(S.cs, S.ct, S.cj);
      // top CAP of (best U cand) = elementwise better of best[i] and
      // cand[CAP-1-i]; staged in registers (two phases, no read/write race)
      double ms[CAP / TK_THREADS];
      uint32_t mt[CAP / TK_THREADS];
      int32_t mj[CAP / TK_THREADS];
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
    const int32_t j = S.bj[i];
    const double v = S.bs[i];
    if (out.final_out) {
      const bool ok = j >= 0 && (!out.positive_only || v > 0.0);
      out.out_idx[static_cast<int64_t>(b) * k + i] = ok ? j : -1;
      out.out_val[static_cast<int64_t>(b) * k + i] = ok ? v : 0.0;
    } else {
      const int64_t at = (static_cast<int64_t>(b) * out.nslices + sl) * k + i;
      out.cs[at] = v;
      out.ct[at] = S.bt[i];
      out.ci[at] = j;
    }
  }
}

template <int CAP>
static int launch_topk(const double* scores, int B, int64_t n, int k, const int32_t* idrank,
                       const int32_t* self_local, int64_t ord_base, int positive_only,
                       int32_t* out_idx, double* out_val, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
  const int smem = sizeof(TopkSmem<CAP>);
  GIFT_CUDA_TRY(cudaFuncSetAttribute(topk_kernel<CAP, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  GIFT_CUDA_TRY(cudaFuncSetAttribute(topk_kernel<CAP, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // slices: enough CTAs to cover the GPU twice, each slice >= 2 * CAP keys
  int64_t nsl = cdiv(2 * sm_count(), B);
  nsl = min64(nsl, cdiv(n, 2 * CAP));
  const size_t per = static_cast<size_t>(B) * k * (8 + 4 + 4);
  if (ws == nullptr || nsl <= 1) nsl = 1;
  while (nsl > 1 && per * nsl + 1024 > ws_bytes) --nsl;
  TopkIn in{};
  in.scores = scores;
  in.n = n;
  in.slice_len = cdiv(n, nsl);
  in.idrank = idrank;
  in.self_local = self_local;
  in.ord_base = ord_base;
  TopkOut out{};
  out.k = k;
  out.positive_only = positive_only;
  out.out_idx = out_idx;
  out.out_val = out_val;
  if (nsl == 1) {
    out.final_out = 1;
    out.nslices = 1;
    topk_kernel<CAP, true><<<dim3(1, B), TK_THREADS, smem, st>>>(in, out);
    GIFT_LAUNCH_CHECK();
    return GIFT_OK;
  }
  Arena ar(ws, ws_bytes);
  const int64_t m = nsl * k;
  double* cs = ar.take<double>(B * m);
  uint32_t* ct = ar.take<uint32_t>(B * m);
  int32_t* ci = ar.take<int32_t>(B * m);
  GIFT_REQUIRE(cs && ct && ci, GIFT_ERR_CAPACITY, "top-k workspace too small");
  out.final_out = 0;
  out.nslices = static_cast<int>(nsl);
  out.cs = cs;
  out.ct = ct;
  out.ci = ci;
  topk_kernel<CAP, true><<<dim3(static_cast<unsigned>(nsl), B), TK_THREADS, smem, st>>>(in, out);
  GIFT_LAUNCH_CHECK();
  TopkIn in2{};
  in2.cs = cs;
  in2.ct = ct;
  in2.ci = ci;
  in2.m = m;
  TopkOut out2 = out;
  out2.final_out = 1;
  out2.nslices = 1;
  topk_kernel<CAP, false><<<dim3(1, B), TK_THREADS, smem, st>>>(in2, out2);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

// Small-k merge of explicit candidate rows (k <= 8): one warp per row.  Each
// lane keeps the sorted best 8 of its strided entries, five xor-shuffle
// merges (merge8) give the row's best 8; same keys and output as topk_kernel.
struct TkKey {
  double s;
  uint32_t t;
  int32_t j;
};
struct TkBetter {
  __device__ bool operator()(const TkKey& x, const TkKey& y) const {
    return key_better(x.s, x.t, y.s, y.t);
  }
};
constexpr int TKS_WARPS = 8;

// WPR = 1: one warp per row (TKS_WARPS rows per CTA); WPR = TKS_WARPS: one CTA
// per row (long rows: the owner reduce's per-warp candidate lists), the warps'
// best-8 lists merged by warp 0 through shared memory.
template <int WPR>
__global__ void __launch_bounds__(TKS_WARPS * 32)
    topk_small_kernel(const TopkIn in, const TopkOut out, int B) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = WPR == 1 ? blockIdx.x * TKS_WARPS + warp : blockIdx.x;
  if (b >= B) return;
  const int64_t e1 = in.counts ? min64(in.m, static_cast<int64_t>(in.counts[b])) : in.m;
  TkKey best[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) best[i] = TkKey{-INFINITY, 0xffffffffu, -1};
  const int64_t row = list_row(in, b);
  const int64_t e0 = WPR == 1 ? lane : warp * 32 + lane;
  for (int64_t e = e0; e < e1; e += 32 * WPR) {
    TkKey x{in.cs[row + e], 0u, in.ci[row + e]};
    if (x.j < 0) continue;
    x.t = in.ct ? in.ct[row + e] : static_cast<uint32_t>(x.j);
    if (!TkBetter()(x, best[7])) continue;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (TkBetter()(x, best[i])) {
        const TkKey t = best[i];
        best[i] = x;
        x = t;
      }
    }
  }
  auto warp_merge = [&]() {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      TkKey oth[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        oth[i].s = __shfl_xor_sync(0xffffffffu, best[i].s, o);
        oth[i].t = __shfl_xor_sync(0xffffffffu, best[i].t, o);
        oth[i].j = __shfl_xor_sync(0xffffffffu, best[i].j, o);
      }
      merge8(best, oth, TkBetter());
    }
  };
  warp_merge();
  if (WPR > 1) {
    __shared__ TkKey s_best[WPR > 1 ? WPR : 1][8];
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < 8; ++i) s_best[warp][i] = best[i];
    __syncthreads();
    if (warp != 0) return;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      best[i] = lane < WPR ? s_best[lane][i] : TkKey{-INFINITY, 0xffffffffu, -1};
    warp_merge();
  }
  const int k = out.k;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (lane == i && i < k) {
      const bool ok = best[i].j >= 0 && (!out.positive_only || best[i].s > 0.0);
      out.out_idx[static_cast<int64_t>(b) * k + i] = ok ? best[i].j : -1;
      out.out_val[static_cast<int64_t>(b) * k + i] = ok ? best[i].s : 0.0;
    }
  }
}

static void launch_topk_small(const TopkIn& in, const TopkOut& out, int B, cudaStream_t st) {
  if (in.m >= 2048)
    topk_small_kernel<TKS_WARPS><<<static_cast<unsigned>(B), TKS_WARPS * 32, 0, st>>>(in, out, B);
  else
    topk_small_kernel<1><<<static_cast<unsigned>(cdiv(B, TKS_WARPS)), TKS_WARPS * 32, 0, st>>>(
        in, out, B);
}

// Best k of explicit (score, tiebreak, global ordinal) rows with per-row
// counts: the merge pass of the dense top-k (used by the sparse S-IF query).
// row_off (optional): row b starts at row_off[b] + b * row_pad, not b * m.
int topk_rows_from_lists(const double* cs, const uint32_t* ct, const int32_t* ci,
                         const int32_t* counts, int32_t B, int64_t m, int32_t k,
                         int32_t positive_only, int32_t* out_idx, double* out_val,
                         cudaStream_t st, const int64_t* row_off, int64_t row_pad) {
  GIFT_REQUIRE(k >= 1 && k <= 256, GIFT_ERR_UNSUPPORTED, "k = %d outside [1, 256]", k);
  if (B <= 0) return GIFT_OK;
  const int smem = sizeof(TopkSmem<256>);
  GIFT_CUDA_TRY(cudaFuncSetAttribute(topk_kernel<256, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  TopkIn in{};
  in.cs = cs;
  in.ct = ct;
  in.ci = ci;
  in.m = m;
  in.counts = counts;
  in.row_off = row_off;
  in.row_pad = row_pad;
  TopkOut out{};
  out.k = k;
  out.positive_only = positive_only;
  out.final_out = 1;
  out.nslices = 1;
  out.out_idx = out_idx;
  out.out_val = out_val;
  if (k <= 8) {
    launch_topk_small(in, out, B, st);
  } else {
    topk_kernel<256, false><<<dim3(1, B), TK_THREADS, smem, st>>>(in, out);
  }
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

}  // namespace gift

using namespace gift;


extern "C" size_t gift_topk_ws_bytes(int32_t B, int64_t n, int32_t k) {
  int64_t nsl = min64(cdiv(2 * 148, max64(B, 1)), cdiv(max64(n, 1), 512));
  return static_cast<size_t>(max64(B, 1)) * k * 16 * max64(nsl, 1) + 4096;
}

extern "C" int gift_topk_rows_ex(const double* scores, int32_t B, int64_t n, int32_t k,
                                 const int32_t* idrank, const int32_t* self_local,
                                 int64_t ord_base, int32_t positive_only, int32_t* out_idx,
                                 double* out_val, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(k >= 1, GIFT_ERR_INVALID, "k must be >= 1");
  GIFT_REQUIRE(k <= 2048, GIFT_ERR_UNSUPPORTED, "k = %d > 2048", k);
  if (B <= 0) return GIFT_OK;
  if (k <= 256) return launch_topk<256>(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx, out_val, ws, ws_bytes, st);
  if (k <= 512) return launch_topk<512>(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx, out_val, ws, ws_bytes, st);
  if (k <= 1024) return launch_topk<1024>(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx, out_val, ws, ws_bytes, st);
  return launch_topk<2048>(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx, out_val, ws, ws_bytes, st);
}

extern "C" int gift_topk_rows(const double* scores, int32_t B, int64_t n, int32_t k,
                              const int32_t* idrank, const int32_t* self_local, int64_t ord_base,
                              int32_t positive_only, int32_t* out_idx, double* out_val,
                              void* stream) {
  return gift_topk_rows_ex(scores, B, n, k, idrank, self_local, ord_base, positive_only, out_idx,
                           out_val, nullptr, 0, stream);
}

extern "C" int gift_topk_cand(const double* cs, const int32_t* ci, int32_t B, int64_t m, int32_t k,
                              int32_t positive_only, int32_t* out_idx, double* out_val,
                              void* stream) {
  return gift_topk_cand_tb(cs, ci, nullptr, B, m, k, positive_only, out_idx, out_val, stream);
}

extern "C" int gift_topk_cand_tb(const double* cs, const int32_t* ci, const uint32_t* ct, int32_t B,
                                 int64_t m, int32_t k, int32_t positive_only, int32_t* out_idx,
                                 double* out_val, void* stream) {
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(k >= 1 && k <= 256, GIFT_ERR_UNSUPPORTED, "k = %d outside [1, 256]", k);
  if (B <= 0) return GIFT_OK;
  const int smem = sizeof(TopkSmem<256>);
  GIFT_CUDA_TRY(cudaFuncSetAttribute(topk_kernel<256, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  TopkIn in{};
  in.cs = cs;
  in.ct = ct;
  in.ci = ci;
  in.m = m;
  TopkOut out{};
  out.k = k;
  out.positive_only = positive_only;
  out.final_out = 1;
  out.nslices = 1;
  out.out_idx = out_idx;
  out.out_val = out_val;
  if (k <= 8) {
    launch_topk_small(in, out, B, st);
  } else {
    topk_kernel<256, false><<<dim3(1, B), TK_THREADS, smem, st>>>(in, out);
  }
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}
