// K2 F-IF build — replaces shapesearch.matching.build_fif (matching.py:106-133).
//
// The reference appends every non-zero view, in shape-major / view-minor
// order, to the list of its nearest codeword.  Here: the quantize key of every
// view (zero views keyed K) is stably radix-sorted (util.cu) giving the
// cell-major permutation; this file gathers the feature rows into that order,
// derives the (cell, shape) segments the scan's max-per-shape runs over, and
// packs segments into scan tiles.
#include "gift_common.cuh"

namespace gift {

// One feature row: copy to the cell-major position (f32/f16 storage and/or
// the tensor-core planes) and return its |x|^2 partial (f64 accumulate).
// Shared by the in-HBM gather and the chunked (streamed) scatter so both
// builds produce bit-identical rows and |p|^2.
template <typename T>
__device__ __forceinline__ double row_emit(const T* __restrict__ in, int d, bool vec,
                                           T* __restrict__ o, __half* __restrict__ hi,
                                           __half* __restrict__ lo) {
  double acc = 0.0;
  constexpr int W = 16 / sizeof(T);
  if (vec) {
    const uint4* in4 = reinterpret_cast<const uint4*>(in);
    for (int k = threadIdx.x; k < d / W; k += blockDim.x) {
      uint4 v = in4[k];
      if (o) reinterpret_cast<uint4*>(o)[k] = v;
      const T* e = reinterpret_cast<const T*>(&v);
      if (hi) {
        if constexpr (sizeof(T) == 4) {
          __half h[W], l[W];
#pragma unroll
          for (int q = 0; q < W; ++q) split2(static_cast<float>(e[q]), h[q], l[q]);
          reinterpret_cast<uint2*>(hi)[k] = *reinterpret_cast<const uint2*>(h);
          if (lo) reinterpret_cast<uint2*>(lo)[k] = *reinterpret_cast<const uint2*>(l);
        } else {
          reinterpret_cast<uint4*>(hi)[k] = v;
        }
      }
#pragma unroll
      for (int q = 0; q < W; ++q) {
        double x = static_cast<double>(static_cast<float>(e[q]));
        acc += x * x;
      }
    }
  } else {
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
      T v = in[k];
      if (o) o[k] = v;
      const float f = static_cast<float>(v);
      if (hi) {
        __half h, l;
        split2(f, h, l);
        hi[k] = sizeof(T) == 4 ? h : __float2half_rn(f);
        if (lo) lo[k] = l;
      }
      double x = static_cast<double>(f);
      acc += x * x;
    }
  }
  return acc;
}

__device__ __forceinline__ float block_sum_f64_to_f32(double acc) {
  __shared__ double red[32];
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
  return static_cast<float>(t);
}

template <typename T>
__global__ void fif_gather_kernel(const T* __restrict__ src, int d, int V,
                                  const uint32_t* __restrict__ perm, int64_t P, int64_t ord_base,
                                  T* __restrict__ out, int32_t* __restrict__ out_ord,
                                  float* __restrict__ out_pn2, bool vec) {
  const int64_t p = blockIdx.x;
  if (p >= P) return;
  const int64_t s = perm[p];
  double acc = row_emit<T>(src + s * d, d, vec, out + p * d, nullptr, nullptr);
  float t = block_sum_f64_to_f32(acc);
  if (threadIdx.x == 0) {
    out_pn2[p] = t;
    out_ord[p] = static_cast<int32_t>(ord_base + s / V);
  }
}

// Streamed build, pass 2: the chunk's view v (global view view_base + v) goes
// to posting pos[v] (< 0: zero view, not stored).
template <typename T>
__global__ void fif_scatter_kernel(const T* __restrict__ src, int d, int V, int64_t nv,
                                   const int32_t* __restrict__ pos, int64_t view_base,
                                   int64_t ord_base, T* __restrict__ out, __half* __restrict__ hi,
                                   __half* __restrict__ lo, int32_t* __restrict__ out_ord,
                                   float* __restrict__ out_pn2, bool vec) {
  const int64_t v = blockIdx.x;
  if (v >= nv) return;
  const int64_t p = pos[view_base + v];
  if (p < 0) return;
  double acc = row_emit<T>(src + v * d, d, vec, out ? out + p * d : nullptr,
                           hi ? hi + p * d : nullptr, lo ? lo + p * d : nullptr);
  float t = block_sum_f64_to_f32(acc);
  if (threadIdx.x == 0) {
    out_pn2[p] = t;
    out_ord[p] = static_cast<int32_t>(ord_base + (view_base + v) / V);
  }
}

__global__ void perm_invert_kernel(const uint32_t* __restrict__ perm, int64_t P,
                                   int32_t* __restrict__ pos) {
  int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < P) pos[perm[p]] = static_cast<int32_t>(p);
}

__device__ __forceinline__ int cell_of(const int64_t* __restrict__ cell_off, int K, int64_t p) {
  // largest c with cell_off[c] <= p
  int lo = 0, hi = K;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (cell_off[mid] <= p)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void seg_flags_kernel(const int64_t* __restrict__ cell_off, const int32_t* __restrict__ ord,
                                 int K, int64_t P, int32_t* __restrict__ flags) {
  int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int c = cell_of(cell_off, K, p);
  flags[p] = (p == cell_off[c] || ord[p] != ord[p - 1]) ? 1 : 0;
}

__global__ void seg_off_kernel(const int64_t* __restrict__ cell_off, const int64_t* __restrict__ sidx,
                               int K, int64_t* __restrict__ seg_off) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > K) return;
  seg_off[c] = sidx[cell_off[c]];
}

__global__ void seg_fill_kernel(const int32_t* __restrict__ flags, const int64_t* __restrict__ sidx,
                                const int32_t* __restrict__ ord, int64_t P,
                                int32_t* __restrict__ seg_ord, int32_t* __restrict__ seg_pstart) {
  int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p > P) return;
  if (p == P) {
    seg_pstart[sidx[P]] = static_cast<int32_t>(P);
    return;
  }
  if (flags[p]) {
    seg_ord[sidx[p]] = ord[p];
    seg_pstart[sidx[p]] = static_cast<int32_t>(p);
  }
}

// Greedy packing of the segments of one cell into tiles of <= tile_n postings.
// emit == false: only count.
__global__ void tiles_kernel(const int64_t* __restrict__ cell_off, const int64_t* __restrict__ seg_off,
                             const int32_t* __restrict__ seg_pstart, int K, int tile_n,
                             int64_t* __restrict__ tile_count_or_off, bool emit,
                             int32_t* __restrict__ t_pstart, int32_t* __restrict__ t_pend,
                             int32_t* __restrict__ t_seg0, int32_t* __restrict__ t_seg1) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K) return;
  const int64_t s_begin = seg_off[c], s_end = seg_off[c + 1];
  const int64_t cell_end = cell_off[c + 1];
  int64_t n = 0;
  int64_t out = emit ? tile_count_or_off[c] : 0;
  auto put = [&](int64_t p0, int64_t p1, int64_t s0, int64_t s1) {
    if (emit) {
      t_pstart[out + n] = static_cast<int32_t>(p0);
      t_pend[out + n] = static_cast<int32_t>(p1);
      t_seg0[out + n] = static_cast<int32_t>(s0);
      t_seg1[out + n] = static_cast<int32_t>(s1);
    }
    ++n;
  };
  if (s_begin == s_end) {
    if (!emit) tile_count_or_off[c] = 0;
    return;
  }
  int64_t cur_start = seg_pstart[s_begin];
  int64_t cur_seg0 = s_begin;
  for (int64_t s = s_begin; s < s_end; ++s) {
    const int64_t a = seg_pstart[s], b = seg_pstart[s + 1];
    if (b - a > tile_n) {
      if (a > cur_start) put(cur_start, a, cur_seg0, s);
      for (int64_t o = a; o < b; o += tile_n) put(o, min64(o + tile_n, b), s, s + 1);
      cur_start = b;
      cur_seg0 = s + 1;
    } else if (b - cur_start > tile_n) {
      put(cur_start, a, cur_seg0, s);
      cur_start = a;
      cur_seg0 = s;
    }
  }
  if (cur_start < cell_end) put(cur_start, cell_end, cur_seg0, s_end);
  if (!emit) tile_count_or_off[c] = n;
}

}  // namespace gift

using namespace gift;

extern "C" int gift_fif_gather(const void* src, int32_t dtype, int32_t d, int32_t V,
                               const uint32_t* perm, int64_t P, int64_t ord_base, void* out_feat,
                               int32_t* out_ord, float* out_pnorm2, void* stream) {
  if (P <= 0) return GIFT_OK;
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(dtype == GIFT_F32 || dtype == GIFT_F16, GIFT_ERR_INVALID,
               "feature storage must be f32 or f16");
  const int threads = d >= 512 ? 256 : 128;
  if (dtype == GIFT_F32) {
    bool vec = d % 4 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
               reinterpret_cast<uintptr_t>(out_feat) % 16 == 0;
    fif_gather_kernel<float><<<static_cast<unsigned>(P), threads, 0, st>>>(
        static_cast<const float*>(src), d, V, perm, P, ord_base, static_cast<float*>(out_feat),
        out_ord, out_pnorm2, vec);
  } else {
    bool vec = d % 8 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
               reinterpret_cast<uintptr_t>(out_feat) % 16 == 0;
    fif_gather_kernel<__half><<<static_cast<unsigned>(P), threads, 0, st>>>(
        static_cast<const __half*>(src), d, V, perm, P, ord_base, static_cast<__half*>(out_feat),
        out_ord, out_pnorm2, vec);
  }
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_perm_invert(const uint32_t* perm, int64_t P, int64_t n_total, int32_t* pos,
                                void* stream) {
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(P <= n_total && n_total < (int64_t(1) << 31), GIFT_ERR_INVALID,
               "perm_invert: sizes out of range");
  if (n_total > 0) GIFT_CUDA_TRY(cudaMemsetAsync(pos, 0xff, sizeof(int32_t) * n_total, st));
  if (P > 0) {
    perm_invert_kernel<<<static_cast<unsigned>(cdiv(P, 256)), 256, 0, st>>>(perm, P, pos);
    GIFT_LAUNCH_CHECK();
  }
  return GIFT_OK;
}

extern "C" int gift_fif_scatter(const void* src, int32_t dtype, int32_t d, int32_t V,
                                int64_t n_views, const int32_t* pos, int64_t view_base,
                                int64_t ord_base, void* out_feat, void* out_hi, void* out_lo,
                                int32_t* out_ord, float* out_pnorm2, void* stream) {
  if (n_views <= 0) return GIFT_OK;
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(dtype == GIFT_F32 || dtype == GIFT_F16, GIFT_ERR_INVALID,
               "feature storage must be f32 or f16");
  GIFT_REQUIRE(out_feat != nullptr || out_hi != nullptr, GIFT_ERR_INVALID,
               "fif_scatter: no feature destination");
  GIFT_REQUIRE(dtype == GIFT_F16 || out_hi == nullptr || out_lo != nullptr, GIFT_ERR_INVALID,
               "fif_scatter: f32 planes need both hi and lo");
  const int threads = d >= 512 ? 256 : 128;
  auto al = [](const void* p) { return p == nullptr || reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  if (dtype == GIFT_F32) {
    bool vec = d % 4 == 0 && al(src) && al(out_feat) && al(out_hi) && al(out_lo) &&
               (out_hi == nullptr || d % 4 == 0);
    fif_scatter_kernel<float><<<static_cast<unsigned>(n_views), threads, 0, st>>>(
        static_cast<const float*>(src), d, V, n_views, pos, view_base, ord_base,
        static_cast<float*>(out_feat), static_cast<__half*>(out_hi), static_cast<__half*>(out_lo),
        out_ord, out_pnorm2, vec);
  } else {
    bool vec = d % 8 == 0 && al(src) && al(out_feat) && al(out_hi);
    fif_scatter_kernel<__half><<<static_cast<unsigned>(n_views), threads, 0, st>>>(
        static_cast<const __half*>(src), d, V, n_views, pos, view_base, ord_base,
        static_cast<__half*>(out_feat), static_cast<__half*>(out_hi), nullptr, out_ord, out_pnorm2,
        vec);
  }
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" size_t gift_fif_build_ws_bytes(int64_t P, int32_t K) {
  return align_up(sizeof(int32_t) * (P + 1), 256) + align_up(sizeof(int64_t) * (P + 2), 256) +
         scan_ws_bytes(P + 1) + align_up(sizeof(int64_t) * (K + 2), 256) + 4096;
}

extern "C" int gift_fif_segments(const int64_t* cell_off, const int32_t* post_ord, int32_t K,
                                 int64_t P, int64_t* seg_off, int32_t* seg_ord,
                                 int32_t* seg_pstart, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  Arena ar(ws, ws_bytes);
  int32_t* flags = ar.take<int32_t>(P + 1);
  int64_t* sidx = ar.take<int64_t>(P + 2);
  GIFT_REQUIRE(flags && sidx, GIFT_ERR_CAPACITY, "segments workspace too small");
  if (P > 0) {
    seg_flags_kernel<<<static_cast<unsigned>(cdiv(P, 256)), 256, 0, st>>>(cell_off, post_ord, K, P,
                                                                          flags);
    GIFT_LAUNCH_CHECK();
  }
  int rc = scan_exclusive_i32_to_i64(flags, sidx, P, true, ar.base + ar.used, ar.remaining(), st);
  if (rc != GIFT_OK) return rc;
  seg_off_kernel<<<static_cast<unsigned>(cdiv(K + 1, 256)), 256, 0, st>>>(cell_off, sidx, K, seg_off);
  GIFT_LAUNCH_CHECK();
  if (seg_ord != nullptr) {
    seg_fill_kernel<<<static_cast<unsigned>(cdiv(P + 1, 256)), 256, 0, st>>>(flags, sidx, post_ord,
                                                                            P, seg_ord, seg_pstart);
    GIFT_LAUNCH_CHECK();
  }
  return GIFT_OK;
}

extern "C" int gift_fif_tiles(const int64_t* cell_off, const int64_t* seg_off,
                              const int32_t* seg_pstart, int32_t K, int32_t tile_n,
                              int64_t* tile_off, int32_t* tile_pstart, int32_t* tile_pend,
                              int32_t* tile_seg0, int32_t* tile_seg1, void* ws, size_t ws_bytes,
                              void* stream) {
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(tile_n >= 1, GIFT_ERR_INVALID, "tile_n must be >= 1");
  Arena ar(ws, ws_bytes);
  int64_t* counts = ar.take<int64_t>(K + 1);
  GIFT_REQUIRE(counts, GIFT_ERR_CAPACITY, "tiles workspace too small");
  tiles_kernel<<<static_cast<unsigned>(cdiv(K, 128)), 128, 0, st>>>(
      cell_off, seg_off, seg_pstart, K, tile_n, counts, false, nullptr, nullptr, nullptr, nullptr);
  GIFT_LAUNCH_CHECK();
  int rc = scan_exclusive_i64(counts, tile_off, K, true, ar.base + ar.used, ar.remaining(), st);
  if (rc != GIFT_OK) return rc;
  if (tile_pstart != nullptr) {
    tiles_kernel<<<static_cast<unsigned>(cdiv(K, 128)), 128, 0, st>>>(
        cell_off, seg_off, seg_pstart, K, tile_n, tile_off, true, tile_pstart, tile_pend,
        tile_seg0, tile_seg1);
    GIFT_LAUNCH_CHECK();
  }
  return GIFT_OK;
}
