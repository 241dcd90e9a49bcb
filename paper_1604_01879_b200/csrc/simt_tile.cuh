// CUDA-core (FFMA) tile mainloop: D[TA x TB] = A[TA x d] . B[TB x d]^T with
// gathered rows, fp32 accumulation in k order (one rounding per FMA, so the
// error bound of a sequential dot product, gamma_d * sum|a_i b_i|, holds —
// the quantize margin relies on it).
//
// Operands are staged by a 3-stage cp.async ring in XOR-swizzled shared
// memory (16-byte chunk c of row r lives at chunk c ^ (r & 7) for fp32 rows,
// c ^ ((r >> 1) & 3) for fp16 rows) so the per-thread 8x4 register tile reads
// conflict-free LDS.128 fragments.  A rows may be fp32 or fp16 (fp16 storage,
// fp32 accumulate); B rows are fp32.
#pragma once
#include "gift_common.cuh"

namespace gift {
namespace simt {

constexpr int TA = 128;  // A rows per tile (postings / views)
constexpr int TB = 64;   // B rows per tile (probes / centroids)
constexpr int BK = 32;   // k elements per stage
constexpr int NSTAGE = 3;
constexpr int NTHR = 256;
constexpr int A_STAGE_BYTES_F32 = TA * BK * 4;  // 16 KB
constexpr int A_STAGE_BYTES_F16 = TA * BK * 2;  //  8 KB
constexpr int B_STAGE_BYTES = TB * BK * 4;      //  8 KB
constexpr int DS_STRIDE = TB + 1;               // epilogue tile stride (floats)

template <bool A_HALF>
struct Cfg {
  static constexpr int A_STAGE = A_HALF ? A_STAGE_BYTES_F16 : A_STAGE_BYTES_F32;
  static constexpr int STAGE = A_STAGE + B_STAGE_BYTES;
  static constexpr int PIPE_BYTES = NSTAGE * STAGE;
  static constexpr int EPI_BYTES = TA * DS_STRIDE * 4;
  static constexpr int SMEM = PIPE_BYTES > EPI_BYTES ? PIPE_BYTES : EPI_BYTES;
};

// Row sources for one tile.  Rows >= na / nb are zero-filled.
struct TileRows {
  const void* a_base;  // element base of A rows (fp32 or fp16)
  const float* b_base;
  int na, nb;
  int d;            // row stride (elements)
  int kbeg = 0;     // k range [kbeg, kend) of this tile (split-k); kend < 0: d
  int kend = -1;
  // row r of A starts at a_base + a_row(r) * d; same for B.
};

// Loads stage (k0) of A and B into shared memory.  vec16 requires d % 4 == 0
// (fp32) / d % 8 == 0 (fp16) and 16-byte aligned bases.
template <bool A_HALF, typename ARowFn, typename BRowFn>
__device__ __forceinline__ void load_stage(char* sA, char* sB, int k0, const TileRows& t,
                                           ARowFn a_row, BRowFn b_row, bool vec16) {
  const int tid = threadIdx.x;
  const int d = t.d;
  const int klim = t.kend < 0 ? d : t.kend;
  if (vec16) {
    if (!A_HALF) {
      // 128 rows x 8 chunks(16B) = 1024 chunk loads, 4 per thread
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int idx = tid + NTHR * j;
        int r = idx >> 3, c = idx & 7;
        int k = k0 + c * 4;
        const float* src = static_cast<const float*>(t.a_base);
        int bytes = 0;
        if (r < t.na && k < klim) {
          src = static_cast<const float*>(t.a_base) + a_row(r) * static_cast<int64_t>(d) + k;
          bytes = min(16, (klim - k) * 4);
        }
        uint32_t dst = smem_u32(sA) + (r * 8 + (c ^ (r & 7))) * 16;
        cp_async16(dst, src, bytes);
      }
    } else {
      // 128 rows x 4 chunks(16B = 8 halves) = 512 loads, 2 per thread
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        int idx = tid + NTHR * j;
        int r = idx >> 2, c = idx & 3;
        int k = k0 + c * 8;
        const __half* src = static_cast<const __half*>(t.a_base);
        int bytes = 0;
        if (r < t.na && k < klim) {
          src = static_cast<const __half*>(t.a_base) + a_row(r) * static_cast<int64_t>(d) + k;
          bytes = min(16, (klim - k) * 2);
        }
        uint32_t dst = smem_u32(sA) + (r * 4 + (c ^ ((r >> 1) & 3))) * 16;
        cp_async16(dst, src, bytes);
      }
    }
    // B: 64 rows x 8 chunks = 512 loads, 2 per thread
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      int idx = tid + NTHR * j;
      int r = idx >> 3, c = idx & 7;
      int k = k0 + c * 4;
      const float* src = t.b_base;
      int bytes = 0;
      if (r < t.nb && k < klim) {
        src = t.b_base + b_row(r) * static_cast<int64_t>(d) + k;
        bytes = min(16, (klim - k) * 4);
      }
      uint32_t dst = smem_u32(sB) + (r * 8 + (c ^ (r & 7))) * 16;
      cp_async16(dst, src, bytes);
    }
  } else {
    // element-wise path for unaligned / odd d (tiny test shapes)
    if (!A_HALF) {
      for (int idx = tid; idx < TA * BK; idx += NTHR) {
        int r = idx / BK, kk = idx % BK, k = k0 + kk;
        const float* src = static_cast<const float*>(t.a_base);
        int bytes = 0;
        if (r < t.na && k < klim) {
          src = static_cast<const float*>(t.a_base) + a_row(r) * static_cast<int64_t>(d) + k;
          bytes = 4;
        }
        uint32_t dst = smem_u32(sA) + (r * 8 + ((kk >> 2) ^ (r & 7))) * 16 + (kk & 3) * 4;
        cp_async4(dst, src, bytes);
      }
    } else {
      // fp16 rows with odd d: plain loads (rare; fp16 storage requires d % 8 == 0)
      for (int idx = tid; idx < TA * BK; idx += NTHR) {
        int r = idx / BK, kk = idx % BK, k = k0 + kk;
        __half v = __float2half(0.f);
        if (r < t.na && k < klim)
          v = static_cast<const __half*>(t.a_base)[a_row(r) * static_cast<int64_t>(d) + k];
        __half* dst = reinterpret_cast<__half*>(sA + (r * 4 + ((kk >> 3) ^ ((r >> 1) & 3))) * 16) +
                      (kk & 7);
        *dst = v;
      }
    }
    for (int idx = tid; idx < TB * BK; idx += NTHR) {
      int r = idx / BK, kk = idx % BK, k = k0 + kk;
      const float* src = t.b_base;
      int bytes = 0;
      if (r < t.nb && k < klim) {
        src = t.b_base + b_row(r) * static_cast<int64_t>(d) + k;
        bytes = 4;
      }
      uint32_t dst = smem_u32(sB) + (r * 8 + ((kk >> 2) ^ (r & 7))) * 16 + (kk & 3) * 4;
      cp_async4(dst, src, bytes);
    }
  }
}

// Thread tile: A rows {wa*32 + i*4 + ag : i<8}, B rows {wb*32 + j*8 + bg : j<4}.
struct Lanes {
  int wa, wb, ag, bg;
  __device__ Lanes() {
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    wa = w & 3;
    wb = w >> 2;
    ag = lane >> 3;
    bg = lane & 7;
  }
  __device__ int a_row(int i) const { return wa * 32 + i * 4 + ag; }
  __device__ int b_row(int j) const { return wb * 32 + j * 8 + bg; }
};

template <bool A_HALF>
__device__ __forceinline__ void compute_stage(const char* sA, const char* sB, const Lanes& L,
                                              float (&acc)[8][4]) {
  if (!A_HALF) {
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) {
      float4 a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int r = L.a_row(i);
        a[i] = *reinterpret_cast<const float4*>(sA + (r * 8 + (kc ^ (r & 7))) * 16);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int r = L.b_row(j);
        b[j] = *reinterpret_cast<const float4*>(sB + (r * 8 + (kc ^ (r & 7))) * 16);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j] = fmaf(a[i].x, b[j].x, acc[i][j]);
          acc[i][j] = fmaf(a[i].y, b[j].y, acc[i][j]);
          acc[i][j] = fmaf(a[i].z, b[j].z, acc[i][j]);
          acc[i][j] = fmaf(a[i].w, b[j].w, acc[i][j]);
        }
    }
  } else {
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      float a[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int r = L.a_row(i);
        uint4 raw = *reinterpret_cast<const uint4*>(sA + (r * 4 + (kc ^ ((r >> 1) & 3))) * 16);
        const __half2* h = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 f = __half22float2(h[q]);
          a[i][2 * q] = f.x;
          a[i][2 * q + 1] = f.y;
        }
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float4 b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int r = L.b_row(j);
          int c = 2 * kc + half;
          b[j] = *reinterpret_cast<const float4*>(sB + (r * 8 + (c ^ (r & 7))) * 16);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[i][j] = fmaf(a[i][4 * half + 0], b[j].x, acc[i][j]);
            acc[i][j] = fmaf(a[i][4 * half + 1], b[j].y, acc[i][j]);
            acc[i][j] = fmaf(a[i][4 * half + 2], b[j].z, acc[i][j]);
            acc[i][j] = fmaf(a[i][4 * half + 3], b[j].w, acc[i][j]);
          }
      }
    }
  }
}

// Full mainloop over d.  smem must hold Cfg<A_HALF>::PIPE_BYTES.
template <bool A_HALF, typename ARowFn, typename BRowFn>
__device__ __forceinline__ void mainloop(char* smem, const TileRows& t, ARowFn a_row,
                                         BRowFn b_row, bool vec16, float (&acc)[8][4]) {
  using C = Cfg<A_HALF>;
  const Lanes L;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const int kb0 = t.kbeg;
  const int nk = ((t.kend < 0 ? t.d : t.kend) - kb0 + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nk) {
      char* base = smem + s * C::STAGE;
      load_stage<A_HALF>(base, base + C::A_STAGE, kb0 + s * BK, t, a_row, b_row, vec16);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    int nxt = kt + NSTAGE - 1;
    if (nxt < nk) {
      char* base = smem + (nxt % NSTAGE) * C::STAGE;
      load_stage<A_HALF>(base, base + C::A_STAGE, kb0 + nxt * BK, t, a_row, b_row, vec16);
    }
    cp_async_commit();
    const char* cur = smem + (kt % NSTAGE) * C::STAGE;
    compute_stage<A_HALF>(cur, cur + C::A_STAGE, L, acc);
  }
  cp_async_wait<0>();
  __syncthreads();
}

}  // namespace simt
}  // namespace gift
