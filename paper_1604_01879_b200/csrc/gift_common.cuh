// Shared helpers for the GIFT sm_100a kernels: error plumbing, cp.async,
// ranking keys, scans.  See include/gift.h for the ABI contract.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gift.h"

namespace gift {

void set_error(const char* fmt, ...);

#define GIFT_CUDA_TRY(expr)                                                  \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      ::gift::set_error("CUDA error '%s' at %s:%d", cudaGetErrorString(e_),  \
                        __FILE__, __LINE__);                                 \
      return GIFT_ERR_CUDA;                                                  \
    }                                                                        \
  } while (0)

#define GIFT_LAUNCH_CHECK() GIFT_CUDA_TRY(cudaGetLastError())

#define GIFT_REQUIRE(cond, code, ...)  \
  do {                                 \
    if (!(cond)) {                     \
      ::gift::set_error(__VA_ARGS__);  \
      return code;                     \
    }                                  \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Arena {
  char* base;
  size_t size;
  size_t used;
  Arena(void* p, size_t n) : base(static_cast<char*>(p)), size(n), used(0) {}
  template <typename T>
  T* take(int64_t count) {
    size_t off = align_up(used, 256);
    size_t bytes = sizeof(T) * static_cast<size_t>(count < 0 ? 0 : count);
    if (off + bytes > size) return nullptr;
    used = off + bytes;
    return reinterpret_cast<T*>(base + off);
  }
  size_t remaining() const { return size > align_up(used, 256) ? size - align_up(used, 256) : 0; }
};

// ------------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(saddr), "l"(g),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ float load_as_f32(const void* p, int dtype, int64_t i) {
  if (dtype == GIFT_F16) return __half2float(static_cast<const __half*>(p)[i]);
  if (dtype == GIFT_F64) return static_cast<float>(static_cast<const double*>(p)[i]);
  return static_cast<const float*>(p)[i];
}
__device__ __forceinline__ double load_as_f64(const void* p, int dtype, int64_t i) {
  if (dtype == GIFT_F16) return static_cast<double>(__half2float(static_cast<const __half*>(p)[i]));
  if (dtype == GIFT_F64) return static_cast<const double*>(p)[i];
  return static_cast<double>(static_cast<const float*>(p)[i]);
}

// Ranking key of the reference's lexsorts: score descending, then a 32-bit
// tiebreak ascending (ordinal for rerank.py:74/:86; (not_self, id rank) for
// index.py:290-294).  Unique per row, so the order is total and deterministic.
struct RankKey {
  double s;
  uint32_t tb;
  int32_t j;
};
__device__ __forceinline__ bool key_better(double s1, uint32_t t1, double s2, uint32_t t2) {
  return s1 > s2 || (s1 == s2 && t1 < t2);
}

// Top-8 of the union of two sorted lists, static indices only (no local
// memory): c[i] = better(a[i], b[7-i]) is bitonic; three half-cleaner stages
// sort it.  `Better(x, y)` is a strict weak order ("x ranks before y").
template <typename T, typename Better>
__device__ __forceinline__ void merge8(T (&a)[8], const T (&b)[8], Better better) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const T y = b[7 - i];
    if (better(y, a[i])) a[i] = y;
  }
#pragma unroll
  for (int stride = 4; stride > 0; stride >>= 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if ((i & stride) == 0) {
        const int j = i + stride;
        if (better(a[j], a[i])) {
          const T t = a[i];
          a[i] = a[j];
          a[j] = t;
        }
      }
    }
  }
}

// Block-wide exclusive scan of one value per thread (blockDim.x <= 1024,
// multiple of 32).  Returns the exclusive prefix; *total receives the sum.
template <typename T>
__device__ T block_exclusive_scan(T v, T* total, T* sbuf /* >= 32 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sbuf[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nwarps ? sbuf[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sbuf[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  T warp_prefix = warp > 0 ? sbuf[warp - 1] : T(0);
  T tot = sbuf[nwarps - 1];
  __syncthreads();
  if (total) *total = tot;
  return warp_prefix + x - v;
}


// ------------------------------------------------------------------------
// tensor-core operand planes: x -> (h1, h2) fp16, x = h1 + 2^-11 h2
// (22 significant bits; the scan and quantize MMAs consume both planes)
// ------------------------------------------------------------------------
constexpr float SPLIT_SCALE = 2048.0f;  // 2^11
__device__ __forceinline__ void split2(float x, __half& h1, __half& h2) {
  h1 = __float2half_rn(x);
  h2 = __float2half_rn((x - __half2float(h1)) * SPLIT_SCALE);
}

// ------------------------------------------------------------------------
// host-side utilities implemented in util.cu
// ------------------------------------------------------------------------
// Exclusive scan of n int64 values (in may alias out).  out[n] = total if
// write_total.  Workspace: scan_ws_bytes(n).
size_t scan_ws_bytes(int64_t n);
int scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, bool write_total, void* ws,
                       size_t ws_bytes, cudaStream_t st);
int scan_exclusive_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, bool write_total,
                              void* ws, size_t ws_bytes, cudaStream_t st);

int sm_count();

// topk.cu: merge pass over explicit candidate rows (score, tiebreak, ordinal)
int topk_rows_from_lists(const double* cs, const uint32_t* ct, const int32_t* ci,
                         const int32_t* counts, int32_t B, int64_t m, int32_t k,
                         int32_t positive_only, int32_t* out_idx, double* out_val,
                         cudaStream_t st, const int64_t* row_off = nullptr,
                         int64_t row_pad = 0);

}  // namespace gift
