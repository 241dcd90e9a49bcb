// K1 quantize — replaces shapesearch.codebook.quantize (codebook.py:111-124).
//
// Reference semantics: d2[c] = sum_k (c_k(f64) - x_k(f64))^2 reduced with
// numpy's pairwise summation (8 accumulators, 128-element leaves, halving
// split rounded to multiples of 8), then argsort(kind="stable")[:ma] — ties
// to the lower centroid index.
//
// Two stages:
//   1. approx[v, c] = |c|^2 - 2 x.c in fp32 on the CUDA-core tile mainloop
//      (simt_tile.cuh);
//   2. per view: T = (ma-th smallest approx) + 2M, where M bounds
//      |approx + |x|^2 - d2_numpy| (fp32 dot error gamma_d |x||c|, rounding of
//      the inputs and of the f64 pairwise sum); every centroid of the true
//      top-ma satisfies approx <= T, so only candidates under T are re-scored
//      with the exact f64 pairwise-order arithmetic (__dsub_rn/__dmul_rn/
//      __dadd_rn, no FMA contraction) and sorted by (d2, index).
// The result is bit-identical to the reference's indices.
#include "fif_scan_tc.cuh"
#include "simt_tile.cuh"

namespace gift {

constexpr int QS_THREADS = 256;
constexpr int QS_LV = 2048;  // leaf sums staged per exact pass (16 KB)
constexpr int QS_WARPS = QS_THREADS / 32;
constexpr int MAX_LEAVES = 256;  // leaves are >= 64 elements -> d <= 16384
constexpr int MAX_K = 8192;
constexpr int MAX_D = 16384;
constexpr int QA_MAX_SPLIT = 8;  // split-k partials of stage 1

template <bool A_HALF>
__global__ void __launch_bounds__(simt::NTHR, 2)
    quant_approx_kernel(const void* __restrict__ X, int64_t n, int d, const float* __restrict__ C,
                        int K, float* __restrict__ part, int ksplit, bool vec16) {
  extern __shared__ __align__(128) char smem[];
  const int64_t v0 = static_cast<int64_t>(blockIdx.x) * simt::TA;
  const int c0 = blockIdx.y * simt::TB;
  simt::TileRows t;
  t.a_base = X;
  t.b_base = C;
  t.na = static_cast<int>(min64(simt::TA, n - v0));
  t.nb = min(simt::TB, K - c0);
  t.d = d;
  // split-k: partial dot over [kbeg, kend) (multiple of BK)
  const int kchunk = ((d + ksplit - 1) / ksplit + simt::BK - 1) / simt::BK * simt::BK;
  t.kbeg = blockIdx.z * kchunk;
  t.kend = min(d, t.kbeg + kchunk);
  float* out = part + static_cast<int64_t>(blockIdx.z) * n * K;
  float acc[8][4];
  simt::mainloop<A_HALF>(
      smem, t, [&](int r) -> int64_t { return v0 + r; }, [&](int r) -> int64_t { return c0 + r; },
      vec16, acc);
  const simt::Lanes L;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int r = L.a_row(i);
    if (r >= t.na) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = L.b_row(j);
      if (c >= t.nb) continue;
      out[(v0 + r) * K + c0 + c] = acc[i][j];
    }
  }
}

__global__ void f64_to_f32_kernel(const double* __restrict__ in, float* __restrict__ out,
                                  int64_t n) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (; i < n; i += stride) out[i] = static_cast<float>(in[i]);
}

struct PairwisePlan {
  int n_leaves, n_ops;
  int leaf_off[MAX_LEAVES];
  int leaf_len[MAX_LEAVES];
  unsigned char ops[2 * MAX_LEAVES];  // 0 = push next leaf, 1 = add top two
};

// Postfix program of numpy's pairwise recursion for a length-d reduction.
__host__ __device__ void build_plan(PairwisePlan& p, int d) {
  struct Frame {
    int off, n, state;
  };
  Frame st[40];
  int top = 0;
  st[0] = {0, d, 0};
  p.n_leaves = 0;
  p.n_ops = 0;
  while (top >= 0) {
    Frame& f = st[top];
    if (f.n <= 128) {
      p.leaf_off[p.n_leaves] = f.off;
      p.leaf_len[p.n_leaves] = f.n;
      p.n_leaves++;
      p.ops[p.n_ops++] = 0;
      --top;
      continue;
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[top + 1] = {f.off, n2, 0};
      ++top;
    } else if (f.state == 1) {
      f.state = 2;
      st[top + 1] = {f.off + n2, f.n - n2, 0};
      ++top;
    } else {
      p.ops[p.n_ops++] = 1;
      --top;
    }
  }
}

__device__ __forceinline__ uint32_t float_order_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float float_from_order_key(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__host__ __device__ __forceinline__ int xpad(int i) { return i + (i >> 7) * 8; }  // bank spread

// Exact numpy-order d2 of candidate centroids, all candidates of a view at
// once: one thread per (candidate, leaf, accumulator) chain.  A leaf of len
// >= 8 elements is 8 interleaved accumulators r_j = sum_s term(off + j + 8s)
// (s < len / 8), combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) -- three
// xor-shuffles over 8 aligned lanes -- plus a sequential tail; a leaf of < 8
// elements is a sequential sum from 0.0.  A chain issues all of its loads
// before its first add (one memory round trip per chain).  Leaf sums land in
// `lvs` [cand][leaf]; the caller combines them with the plan's postfix
// program.  Must be called by all threads of the CTA (warp-uniform trip
// count; returns after a __syncthreads).
template <int NTHR>
__device__ void exact_leaves(const float* __restrict__ xs, const void* X, int xdtype, int64_t xoff,
                             const float* __restrict__ C, int d, const int* ci, int q0, int nq,
                             const PairwisePlan& plan, double* lvs) {
  const int tid = threadIdx.x;
  const int nch = plan.n_leaves * 8;
  const int units = nq * nch;
  auto xat = [&](int k) -> double {
    return xs ? static_cast<double>(xs[xpad(k)]) : load_as_f64(X, xdtype, xoff + k);
  };
  auto sq = [](double c, double x) {
    const double t = __dsub_rn(c, x);
    return __dmul_rn(t, t);
  };
  for (int u0 = 0; u0 < units; u0 += NTHR) {
    const int u = u0 + tid;
    const bool act = u < units;
    const int q = act ? u / nch : 0;
    const int rem = u - q * nch;
    const int l = rem >> 3, j = rem & 7;
    const int off = act ? plan.leaf_off[l] : 0, len = act ? plan.leaf_len[l] : 0;
    const int lim = len - len % 8;
    const float* crow = C + static_cast<int64_t>(ci[q0 + q]) * d;
    double r = 0.0;
    if (act && len >= 8) {
      double xv[16];
      float cv[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const bool ok = 8 * s < lim;
        xv[s] = ok ? xat(off + j + 8 * s) : 0.0;
        cv[s] = ok ? crow[off + j + 8 * s] : 0.f;
      }
      r = sq(static_cast<double>(cv[0]), xv[0]);
#pragma unroll
      for (int s = 1; s < 16; ++s)
        if (8 * s < lim) r = __dadd_rn(r, sq(static_cast<double>(cv[s]), xv[s]));
    }
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (act && j == 0) {
      if (len < 8) {
        r = 0.0;
        for (int i = 0; i < len; ++i) r = __dadd_rn(r, sq(static_cast<double>(crow[off + i]), xat(off + i)));
      } else {
        for (int i = lim; i < len; ++i)
          r = __dadd_rn(r, sq(static_cast<double>(crow[off + i]), xat(off + i)));
      }
      lvs[q * plan.n_leaves + l] = r;
    }
  }
  __syncthreads();
}

// Postfix program of the pairwise recursion over one candidate's leaf sums.
__device__ double combine_leaves(const PairwisePlan& plan, const double* lv) {
  double stk[24];
  int sp = 0, li = 0;
  for (int o = 0; o < plan.n_ops; ++o) {
    if (plan.ops[o] == 0) {
      stk[sp++] = lv[li++];
    } else {
      const double bb = stk[--sp];
      const double aa = stk[--sp];
      stk[sp++] = __dadd_rn(aa, bb);
    }
  }
  return stk[0];
}

__global__ void __launch_bounds__(QS_THREADS)
    quant_select_kernel(const float* __restrict__ approx, int64_t n, int K, int ma,
                        const void* __restrict__ X, int xdtype, int d, const float* __restrict__ C,
                        double cmax, const uint8_t* __restrict__ nz, int zero_key, int p2k,
                        int need_order, int stage_x, int32_t* __restrict__ out,
                        const double* __restrict__ cn2, int ksplit, double dot_eps,
                        const int32_t* __restrict__ list,
                        const int32_t* __restrict__ list_count,
                        const __grid_constant__ PairwisePlan plan) {
  extern __shared__ __align__(128) char smem[];
  float* a = reinterpret_cast<float*>(smem);
  double* cd = reinterpret_cast<double*>(smem + ((K * 4 + 15) / 16) * 16);
  int* ci = reinterpret_cast<int*>(cd + p2k);
  float* xs = stage_x ? reinterpret_cast<float*>(ci + p2k) : nullptr;
  __shared__ double lvs[QS_LV];
  __shared__ unsigned hist[256];
  __shared__ double s_red[QS_WARPS];
  __shared__ float s_redf[QS_WARPS];
  __shared__ float s_small[QS_WARPS][8];
  __shared__ uint32_t s_prefix;
  __shared__ int s_rank, s_nc;
  __shared__ float s_kth;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // persistent CTAs over the views the warp kernel left (all views without it)
  const int64_t total = list != nullptr ? static_cast<int64_t>(*list_count) : n;
  auto one = [&](const int64_t v) {
  if (nz != nullptr && nz[v] == 0) {
    for (int s = tid; s < ma; s += QS_THREADS) out[v * ma + s] = zero_key >= 0 ? zero_key : -1;
    return;
  }
  const int64_t xoff = v * static_cast<int64_t>(d);
  // stage x (exact in f32 for f32/f16 inputs) and |x| (f64) for the margin
  double xsq = 0.0;
  const float* xf = static_cast<const float*>(X) + xoff;
  if (xs != nullptr && xdtype == GIFT_F32 && (d & 3) == 0 &&
      (reinterpret_cast<uintptr_t>(xf) & 15) == 0) {
    const int d4 = d >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(xf);
    for (int k0 = tid; k0 < d4; k0 += 4 * QS_THREADS) {
      float4 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u * QS_THREADS;
        t[u] = k < d4 ? x4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u * QS_THREADS;
        if (k < d4) {
          float* dst = xs + xpad(4 * k);
          dst[0] = t[u].x;
          dst[1] = t[u].y;
          dst[2] = t[u].z;
          dst[3] = t[u].w;
          xsq += static_cast<double>(t[u].x) * t[u].x + static_cast<double>(t[u].y) * t[u].y +
                 static_cast<double>(t[u].z) * t[u].z + static_cast<double>(t[u].w) * t[u].w;
        }
      }
    }
  } else {
    for (int k = tid; k < d; k += QS_THREADS) {
      const double xv = load_as_f64(X, xdtype, xoff + k);
      if (xs) xs[xpad(k)] = static_cast<float>(xv);
      xsq += xv * xv;
    }
  }
  for (int o = 16; o > 0; o >>= 1) xsq += __shfl_xor_sync(0xffffffffu, xsq, o);
  if (lane == 0) s_red[warp] = xsq;
  for (int c = tid; c < K; c += QS_THREADS) {
    float pz[QA_MAX_SPLIT];
#pragma unroll
    for (int z = 0; z < QA_MAX_SPLIT; ++z)
      pz[z] = z < ksplit ? approx[static_cast<int64_t>(z) * n * K + v * K + c] : 0.f;
    float dot = pz[0];
#pragma unroll
    for (int z = 1; z < QA_MAX_SPLIT; ++z)
      if (z < ksplit) dot += pz[z];
    a[c] = static_cast<float>(cn2[c]) - 2.0f * dot;
  }
  if (tid == 0) s_nc = 0;
  __syncthreads();
  double xn2 = 0.0;
  for (int w = 0; w < QS_WARPS; ++w) xn2 += s_red[w];
  const double xn = sqrt(xn2) * (1.0 + 1e-6) + 1e-300;

  // ma-th smallest approx value
  if (ma == 1) {
    float m = INFINITY;
    for (int c = tid; c < K; c += QS_THREADS) m = fminf(m, a[c]);
    for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_redf[warp] = m;
    __syncthreads();
    if (tid == 0) {
      float mm = INFINITY;
      for (int w = 0; w < QS_WARPS; ++w) mm = fminf(mm, s_redf[w]);
      s_kth = mm;
    }
    __syncthreads();
  } else if (ma <= 8) {
    // per-thread sorted lists, shuffle merges, final merge of the 4 warps
    float loc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) loc[i] = INFINITY;
    for (int c = tid; c < K; c += QS_THREADS) {
      float x = a[c];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < ma && x < loc[i]) {
          float t = loc[i];
          loc[i] = x;
          x = t;
        }
      }
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      float oth[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) oth[i] = __shfl_xor_sync(0xffffffffu, loc[i], o);
      merge8(loc, oth, [](float x, float y) { return x < y; });
    }
    if (lane == 0)
      for (int i = 0; i < 8; ++i) s_small[warp][i] = loc[i];
    __syncthreads();
    if (tid == 0) {
      float all[QS_WARPS * 8];
      for (int w = 0; w < QS_WARPS; ++w)
        for (int i = 0; i < 8; ++i) all[w * 8 + i] = s_small[w][i];
      for (int i = 0; i < ma; ++i) {
        int best = i;
        for (int j = i + 1; j < QS_WARPS * 8; ++j)
          if (all[j] < all[best]) best = j;
        const float t = all[i];
        all[i] = all[best];
        all[best] = t;
      }
      s_kth = all[ma - 1];
    }
    __syncthreads();
  } else {
    // radix select (large ma)
    if (tid == 0) {
      s_prefix = 0;
      s_rank = ma - 1;
    }
    uint32_t mask = 0;
    for (int pass = 3; pass >= 0; --pass) {
      const int shift = 8 * pass;
      for (int b = tid; b < 256; b += QS_THREADS) hist[b] = 0;
      __syncthreads();
      const uint32_t prefix = s_prefix;
      for (int c = tid; c < K; c += QS_THREADS) {
        uint32_t u = float_order_key(a[c]);
        if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        int rank = s_rank;
        unsigned cum = 0;
        for (int b = 0; b < 256; ++b) {
          if (cum + hist[b] > static_cast<unsigned>(rank)) {
            s_prefix = prefix | (static_cast<uint32_t>(b) << shift);
            s_rank = rank - static_cast<int>(cum);
            break;
          }
          cum += hist[b];
        }
      }
      mask |= 255u << shift;
      __syncthreads();
    }
    if (tid == 0) s_kth = float_from_order_key(s_prefix);
    __syncthreads();
  }

  // rigorous margin M >= |approx + |x|^2 - d2_numpy|
  const double u32 = 5.9604644775390625e-08;  // 2^-24
  const double u64 = 1.1102230246251565e-16;  // 2^-53
  // dot_eps bounds |fl(x.c) - x.c| / (|x| |c|) of stage 1 (CUDA-core split-k
  // chains: gamma of the chunk length + partial additions; tensor cores:
  // tc_dot_eps)
  const double M = 1.5 * (2.0 * dot_eps * xn * cmax + 3.0 * u32 * cmax * cmax +
                          2.0 * u32 * xn * cmax + (d + 4) * u64 * (xn + cmax) * (xn + cmax)) +
                   1e-30;
  const double thresh = static_cast<double>(s_kth) + 2.0 * M;
  for (int c = tid; c < K; c += QS_THREADS) {
    if (static_cast<double>(a[c]) <= thresh) {
      int pos = atomicAdd(&s_nc, 1);
      ci[pos] = c;
    }
  }
  __syncthreads();
  const int nc = s_nc;
  if (nc == ma && (ma == 1 || !need_order)) {
    // the candidate set is the answer; only its order would need exact d2
    if (tid == 0) {
      for (int i = 1; i < ma; ++i)  // ascending index: deterministic slot order
        for (int j = i; j > 0 && ci[j] < ci[j - 1]; --j) {
          const int t = ci[j];
          ci[j] = ci[j - 1];
          ci[j - 1] = t;
        }
      for (int s = 0; s < ma; ++s) out[v * ma + s] = ci[s];
    }
    return;
  }
  // exact numpy-order d2 of every candidate, QS_LV / n_leaves candidates per
  // pass
  const int per = QS_LV / plan.n_leaves;
  for (int q0 = 0; q0 < nc; q0 += per) {
    const int nq = min(per, nc - q0);
    exact_leaves<QS_THREADS>(xs, X, xdtype, xoff, C, d, ci, q0, nq, plan, lvs);
    for (int q = tid; q < nq; q += QS_THREADS) cd[q0 + q] = combine_leaves(plan, lvs + q * plan.n_leaves);
    __syncthreads();
  }
  // ascending (d2, index): bitonic over the next power of 2
  int p2 = 1;
  while (p2 < nc) p2 <<= 1;
  for (int i = nc + tid; i < p2; i += QS_THREADS) {
    cd[i] = INFINITY;
    ci[i] = 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < (p2 >> 1); i += QS_THREADS) {
        const int lo = 2 * stride * (i / stride) + (i % stride);
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const double dl = cd[lo], dh = cd[hi];
        const int il = ci[lo], ih = ci[hi];
        const bool hi_first = (dh < dl) || (dh == dl && ih < il);
        if (hi_first == up) {
          cd[lo] = dh;
          cd[hi] = dl;
          ci[lo] = ih;
          ci[hi] = il;
        }
      }
      __syncthreads();
    }
  }
  for (int s = tid; s < ma; s += QS_THREADS) out[v * ma + s] = ci[s];
  };
  for (int64_t i = blockIdx.x; i < total; i += gridDim.x) {
    one(list != nullptr ? static_cast<int64_t>(list[i]) : i);
    __syncthreads();
  }
}


// Fast path of stage 2 (ma <= 8): one warp per vector.  Pass 1 finds the
// ma-th smallest approx value (per-lane sorted lists + xor-shuffle merges),
// pass 2 collects the candidates under the margin with a ballot; unambiguous
// sets are written directly, every other view is flagged for the exact
// re-check of the CTA-per-vector kernel above (a few percent of the views).
constexpr int QW_WARPS = 8;

__global__ void __launch_bounds__(QW_WARPS * 32)
    quant_select_warp_kernel(const float* __restrict__ approx, int64_t n, int K, int ma,
                             const void* __restrict__ X, int xdtype, int d,
                             const float* __restrict__ C, double cmax,
                             const uint8_t* __restrict__ nz, int zero_key, int need_order,
                             int32_t* __restrict__ out, const double* __restrict__ cn2,
                             int ksplit, double dot_eps, const float* __restrict__ xnorm2,
                             int32_t* __restrict__ list, int32_t* __restrict__ list_count) {
  __shared__ int s_ci[QW_WARPS][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t v = static_cast<int64_t>(blockIdx.x) * QW_WARPS + warp;
  if (v >= n) return;
  if (nz != nullptr && nz[v] == 0) {
    for (int s = lane; s < ma; s += 32) out[v * ma + s] = zero_key >= 0 ? zero_key : -1;
    return;
  }
  const int64_t xoff = v * static_cast<int64_t>(d);
  double xn;
  if (xnorm2 != nullptr) {
    xn = sqrt(static_cast<double>(xnorm2[v])) * (1.0 + 1e-5) + 1e-300;
  } else {
    double xsq = 0.0;
    for (int k = lane; k < d; k += 32) {
      const double xv = load_as_f64(X, xdtype, xoff + k);
      xsq += xv * xv;
    }
    for (int o = 16; o > 0; o >>= 1) xsq += __shfl_xor_sync(0xffffffffu, xsq, o);
    xn = sqrt(xsq) * (1.0 + 1e-6) + 1e-300;
  }
  auto approx_at = [&](int c) -> float {
    float dot = approx[v * K + c];
    for (int z = 1; z < ksplit; ++z) dot += approx[static_cast<int64_t>(z) * n * K + v * K + c];
    return static_cast<float>(cn2[c]) - 2.0f * dot;
  };
  // pass 1: ma-th smallest.  For K <= 512 the row stays in registers (all
  // loads issued up front); larger codebooks re-read it in pass 2.
  constexpr int QW_REG = 16;
  const bool in_regs = K <= 32 * QW_REG;
  float av[QW_REG];
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < QW_REG; ++i) {
      const int c = lane + 32 * i;
      av[i] = c < K ? approx[v * K + c] : 0.f;
    }
    for (int z = 1; z < ksplit; ++z) {
#pragma unroll
      for (int i = 0; i < QW_REG; ++i) {
        const int c = lane + 32 * i;
        if (c < K) av[i] += approx[static_cast<int64_t>(z) * n * K + v * K + c];
      }
    }
#pragma unroll
    for (int i = 0; i < QW_REG; ++i) {
      const int c = lane + 32 * i;
      av[i] = c < K ? static_cast<float>(cn2[c]) - 2.0f * av[i] : INFINITY;
    }
  }
  float loc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) loc[i] = INFINITY;
  auto insert = [&](float x) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < ma && x < loc[i]) {
        const float t = loc[i];
        loc[i] = x;
        x = t;
      }
    }
  };
  // large codebooks: QW_UNR row values per lane loaded before they are
  // inserted (memory-level parallelism; the row is re-read in pass 2)
  constexpr int QW_UNR = 8;
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < QW_REG; ++i) insert(av[i]);
  } else {
    for (int c0 = lane; c0 < K; c0 += 32 * QW_UNR) {
      float xs[QW_UNR];
#pragma unroll
      for (int u = 0; u < QW_UNR; ++u) {
        const int c = c0 + 32 * u;
        xs[u] = c < K ? approx_at(c) : INFINITY;
      }
#pragma unroll
      for (int u = 0; u < QW_UNR; ++u) insert(xs[u]);
    }
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    float oth[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) oth[i] = __shfl_xor_sync(0xffffffffu, loc[i], o);
    merge8(loc, oth, [](float x, float y) { return x < y; });
  }
  float kth = loc[0];
#pragma unroll
  for (int i = 1; i < 8; ++i)
    if (i == ma - 1) kth = loc[i];
  const double u32 = 0x1p-24, u64 = 0x1p-53;
  const double M = 1.5 * (2.0 * dot_eps * xn * cmax + 3.0 * u32 * cmax * cmax +
                          2.0 * u32 * xn * cmax + (d + 4) * u64 * (xn + cmax) * (xn + cmax)) +
                   1e-30;
  const double thresh = static_cast<double>(kth) + 2.0 * M;
  // pass 2: candidates under the threshold
  int cnt = 0;
  const unsigned lt = (1u << lane) - 1u;
  auto collect = [&](int c, float x) {  // warp-uniform call
    const bool hit = c < K && static_cast<double>(x) <= thresh;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    const int pos = cnt + __popc(bal & lt);
    if (hit && pos < 8) s_ci[warp][pos] = c;
    cnt += __popc(bal);
  };
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < QW_REG; ++i) collect(lane + 32 * i, av[i]);
  } else {
    for (int b0 = 0; b0 < K; b0 += 32 * QW_UNR) {
      float xs[QW_UNR];
#pragma unroll
      for (int u = 0; u < QW_UNR; ++u) {
        const int c = b0 + 32 * u + lane;
        xs[u] = c < K ? approx_at(c) : INFINITY;
      }
#pragma unroll
      for (int u = 0; u < QW_UNR; ++u) collect(b0 + 32 * u + lane, xs[u]);
    }
  }
  __syncwarp();
  int* ci = s_ci[warp];
  if (cnt == ma && (ma == 1 || !need_order)) {
    if (lane == 0) {
      for (int i = 1; i < ma; ++i)
        for (int j = i; j > 0 && ci[j] < ci[j - 1]; --j) {
          const int t = ci[j];
          ci[j] = ci[j - 1];
          ci[j - 1] = t;
        }
      for (int s = 0; s < ma; ++s) out[v * ma + s] = ci[s];
    }
    return;
  }
  if (lane == 0) list[atomicAdd(list_count, 1)] = static_cast<int32_t>(v);  // exact re-check
}

}  // namespace gift

using namespace gift;

static size_t quant_fixed_bytes(int d, int K) {
  return 2 * align_up(static_cast<size_t>(K) * d * 2, 1024) + 16384;
}
static size_t quant_row_bytes(int d, int K) {
  // partials + (f64 -> f32 conversion | two fp16 planes)
  return static_cast<size_t>(K) * 4 * QA_MAX_SPLIT + static_cast<size_t>(d) * 4 + 64;
}

static int64_t quant_rows_for(size_t ws_bytes, int d, int K, int xdtype) {
  (void)xdtype;
  const size_t fixed = quant_fixed_bytes(d, K);
  if (ws_bytes < fixed) return 0;
  return static_cast<int64_t>((ws_bytes - fixed) / quant_row_bytes(d, K));
}

extern "C" size_t gift_quantize_ws_bytes(int64_t n, int32_t d, int32_t K, int32_t xdtype) {
  (void)xdtype;
  int64_t rows = n < 16384 ? (n < 128 ? 128 : n) : 16384;
  return quant_row_bytes(d, K) * rows + quant_fixed_bytes(d, K) + 4096;
}

namespace gift {
int quantize_impl(const void* X, int32_t xdtype, int64_t n, int32_t d, const float* C,
                  const double* cnorm2, int32_t K, double cmax_norm, int32_t ma,
                  const uint8_t* nz, int32_t zero_key, int32_t* out_idx, void* ws,
                  size_t ws_bytes, void* stream, bool need_order, const float* xnorm2,
                  bool allow_tc) {
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(K >= 1 && d >= 1, GIFT_ERR_EMPTY, "empty codebook");
  GIFT_REQUIRE(ma >= 1 && ma <= K, GIFT_ERR_INVALID, "ma must be in [1, %d]", K);
  GIFT_REQUIRE(K <= MAX_K, GIFT_ERR_UNSUPPORTED, "codebook size %d > %d", K, MAX_K);
  GIFT_REQUIRE(d <= MAX_D, GIFT_ERR_UNSUPPORTED, "dimension %d > %d", d, MAX_D);
  GIFT_REQUIRE(xdtype == GIFT_F32 || xdtype == GIFT_F16 || xdtype == GIFT_F64, GIFT_ERR_INVALID,
               "bad dtype");
  if (n <= 0) return GIFT_OK;
  int64_t rows = quant_rows_for(ws_bytes, d, K, xdtype);
  if (rows >= n) rows = n;
  else rows = rows / simt::TA * simt::TA;
  GIFT_REQUIRE(rows >= 1, GIFT_ERR_CAPACITY, "quantize workspace too small");

  int p2k = 1;
  while (p2k < K) p2k <<= 1;
  const int stage_x = (xdtype != GIFT_F64) ? 1 : 0;
  const size_t sel_smem = ((static_cast<size_t>(K) * 4 + 15) / 16) * 16 +
                          static_cast<size_t>(p2k) * 12 +
                          (stage_x ? static_cast<size_t>(xpad(d) + 16) * 4 : 0);
  GIFT_CUDA_TRY(cudaFuncSetAttribute(quant_select_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sel_smem)));
  PairwisePlan plan;
  build_plan(plan, d);
  const bool a_half = xdtype == GIFT_F16;
  const int approx_smem = a_half ? simt::Cfg<true>::SMEM : simt::Cfg<false>::SMEM;
  if (a_half)
    GIFT_CUDA_TRY(cudaFuncSetAttribute(quant_approx_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, approx_smem));
  else
    GIFT_CUDA_TRY(cudaFuncSetAttribute(quant_approx_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, approx_smem));

  Arena ar(ws, ws_bytes);
  float* approx = ar.take<float>(rows * K * QA_MAX_SPLIT);
  float* xconv = xdtype == GIFT_F64 ? ar.take<float>(rows * static_cast<int64_t>(d)) : nullptr;
  GIFT_REQUIRE(approx != nullptr && (xdtype != GIFT_F64 || xconv != nullptr), GIFT_ERR_CAPACITY,
               "quantize workspace too small");
  const bool use_tc = allow_tc && quant_tc_supported(d, xdtype);
  // views left for the CTA kernel by the warp kernel (+ their count)
  int32_t* list = ma <= 8 ? ar.take<int32_t>(rows + 1) : nullptr;
  GIFT_REQUIRE(ma > 8 || list != nullptr, GIFT_ERR_CAPACITY, "quantize workspace too small");
  int32_t* list_count = list != nullptr ? list + rows : nullptr;
  const int sel_grid = sm_count() * 4;
  void* tc_ws = ar.base + align_up(ar.used, 256);
  const size_t tc_ws_bytes = ar.remaining();

  const size_t esz = xdtype == GIFT_F16 ? 2 : (xdtype == GIFT_F64 ? 8 : 4);
  for (int64_t r0 = 0; r0 < n; r0 += rows) {
    const int64_t nr = min64(rows, n - r0);
    const char* xs = static_cast<const char*>(X) + r0 * d * esz;
    const void* a_src = xs;
    if (xdtype == GIFT_F64) {
      int64_t cnt = nr * d;
      f64_to_f32_kernel<<<static_cast<unsigned>(min64(cdiv(cnt, 256), 4096)), 256, 0, st>>>(
          reinterpret_cast<const double*>(xs), xconv, cnt);
      GIFT_LAUNCH_CHECK();
      a_src = xconv;
    }
    int ksplit = 1;
    double dot_eps;
    if (use_tc) {
      int rc = quant_approx_tc(xs, xdtype, nr, d, C, K, approx, QA_MAX_SPLIT, &ksplit, tc_ws,
                               tc_ws_bytes, st);
      if (rc) return rc;
      dot_eps = tc_dot_eps(d);
    } else {
      const bool aligned = (reinterpret_cast<uintptr_t>(a_src) % 16 == 0) &&
                           (reinterpret_cast<uintptr_t>(C) % 16 == 0);
      const bool vec16 = aligned && (a_half ? (d % 8 == 0) : (d % 4 == 0));
      // split-k so the grid covers the GPU ~2x (2 CTAs/SM), chunks >= 512
      const int64_t tiles = cdiv(nr, simt::TA) * cdiv(K, simt::TB);
      ksplit = static_cast<int>(min64(cdiv(4 * sm_count(), tiles), QA_MAX_SPLIT));
      ksplit = static_cast<int>(max64(1, min64(ksplit, d / 512)));
      const int kchunk = ((d + ksplit - 1) / ksplit + simt::BK - 1) / simt::BK * simt::BK;
      ksplit = (d + kchunk - 1) / kchunk;
      dim3 grid(static_cast<unsigned>(cdiv(nr, simt::TA)), static_cast<unsigned>(cdiv(K, simt::TB)),
                static_cast<unsigned>(ksplit));
      if (a_half)
        quant_approx_kernel<true><<<grid, simt::NTHR, approx_smem, st>>>(a_src, nr, d, C, K, approx,
                                                                        ksplit, vec16);
      else
        quant_approx_kernel<false><<<grid, simt::NTHR, approx_smem, st>>>(a_src, nr, d, C, K,
                                                                         approx, ksplit, vec16);
      GIFT_LAUNCH_CHECK();
      // sequential fp32 FMA chain of kchunk terms + (ksplit - 1) partial adds
      const double u32 = 0x1p-24;
      const double m = kchunk + ksplit + 2;
      dot_eps = m * u32 / (1.0 - m * u32) + 2.0 * u32;
    }
    if (list != nullptr) {
      GIFT_CUDA_TRY(cudaMemsetAsync(list_count, 0, sizeof(int32_t), st));
      quant_select_warp_kernel<<<static_cast<unsigned>(cdiv(nr, QW_WARPS)), QW_WARPS * 32, 0,
                                 st>>>(approx, nr, K, ma, xs, xdtype, d, C, cmax_norm,
                                       nz ? nz + r0 : nullptr, zero_key, need_order ? 1 : 0,
                                       out_idx + r0 * ma, cnorm2, ksplit, dot_eps,
                                       xnorm2 ? xnorm2 + r0 : nullptr, list, list_count);
      GIFT_LAUNCH_CHECK();
    }
    quant_select_kernel<<<static_cast<unsigned>(min64(nr, sel_grid)), QS_THREADS, sel_smem, st>>>(
        approx, nr, K, ma, xs, xdtype, d, C, cmax_norm, nz ? nz + r0 : nullptr, zero_key, p2k,
        need_order ? 1 : 0, stage_x, out_idx + r0 * ma, cnorm2, ksplit, dot_eps, list, list_count,
        plan);
    GIFT_LAUNCH_CHECK();
  }
  return GIFT_OK;
}
}  // namespace gift

extern "C" int gift_quantize(const void* X, int32_t xdtype, int64_t n, int32_t d, const float* C,
                             const double* cnorm2, int32_t K, double cmax_norm, int32_t ma,
                             const uint8_t* nz, int32_t zero_key, int32_t* out_idx, void* ws,
                             size_t ws_bytes, void* stream) {
  return gift_quantize_ex(X, xdtype, n, d, C, cnorm2, K, cmax_norm, ma, nz, zero_key, out_idx, ws,
                          ws_bytes, 0, stream);
}

extern "C" int gift_quantize_ex(const void* X, int32_t xdtype, int64_t n, int32_t d,
                                const float* C, const double* cnorm2, int32_t K,
                                double cmax_norm, int32_t ma, const uint8_t* nz,
                                int32_t zero_key, int32_t* out_idx, void* ws, size_t ws_bytes,
                                int32_t flags, void* stream) {
  GIFT_REQUIRE((flags & ~GIFT_QUANT_SIMT) == 0, GIFT_ERR_INVALID, "unknown quantize flags 0x%x",
               flags);
  return quantize_impl(X, xdtype, n, d, C, cnorm2, K, cmax_norm, ma, nz, zero_key, out_idx, ws,
                       ws_bytes, stream, true, nullptr, !(flags & GIFT_QUANT_SIMT));
}
