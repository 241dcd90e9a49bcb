// K3 F-IF score — replaces shapesearch.matching.query_fif (matching.py:136-161)
// for a whole batch of queries at once.
//
// Reference (per query, per non-zero view q_i):
//   view_best[p] = max over the postings of shape p stored in the ma nearest
//                  cells of q_i of clip(q_i . f, 0, 1)            (:152-159)
//   total += view_best ; score = total / Vq                       (:160-161)
//
// Batched, cell-major plan (one pass over each probed cell per batch):
//   plan   : every (query view, ma slot) probe is bucketed by cell;
//   scan   : persistent CTAs take work items (posting tile of a cell x tile of
//            that cell's probes), compute the posting x probe dot tile on the
//            CUDA-core mainloop, and reduce each (cell, shape) segment of the
//            tile to its maximum similarity -> compact[cell][probe][segment];
//   reduce : per (query, range of shapes): max over the ma slots of a view,
//            f64 sum over the views in view order, / Vq  -> dense scores.
// Deterministic: no floating-point atomics; the only atomics are integer
// counters and atomicMax on non-negative float bits (order-independent).
#include <stdlib.h>

#include "fif_scan_tc.cuh"
#include "simt_tile.cuh"

namespace gift {

constexpr int64_t RED_SMEM = 64 * 1024;  // reduce CTA view-best tile budget
constexpr int RED_THREADS = 256;
constexpr int RED_MAX_RS = 2048;  // shapes per reduce range (reduce_rs cap)
constexpr int PLAN_THREADS = 1024;


__global__ void probe_count_kernel(const int32_t* __restrict__ cells, int64_t nprobes,
                                   int32_t* __restrict__ counts) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nprobes) return;
  int c = cells[i];
  if (c >= 0) atomicAdd(&counts[c], 1);
}

__global__ void __launch_bounds__(PLAN_THREADS)
    probe_plan_kernel(const int32_t* __restrict__ counts, int K, const int64_t* __restrict__ seg_off,
                      const int64_t* __restrict__ tile_off, int32_t* __restrict__ probe_off,
                      int64_t* __restrict__ outbase, int64_t* __restrict__ item_off,
                      int32_t* __restrict__ cursor, int64_t* __restrict__ meta, int64_t capacity,
                      int ptile, int tile_div, int dense_min, int64_t* __restrict__ item_off2) {
  __shared__ int64_t sbuf[32];
  const int per = (K + PLAN_THREADS - 1) / PLAN_THREADS;
  const int c0 = threadIdx.x * per;
  // dense cells (>= dense_min probes, fp16-exact batch: meta[M_QLO] from
  // query_lo_kernel) go to the probe-major scan's list (fif_scan_dense.cu):
  // ceil(T / 2) posting tile pairs x ceil(n / 256) probe tiles
  const bool split = dense_min > 0 && meta[M_QLO] == 0;
  auto items = [&](int64_t n, int64_t T, int64_t& i1, int64_t& i2) {
    const bool dn = split && n >= dense_min;
    i1 = dn ? 0 : (T + tile_div - 1) / tile_div * ((n + ptile - 1) / ptile);
    i2 = dn ? (T + 1) / 2 * ((n + 255) / 256) : 0;
  };
  int64_t s_cnt = 0, s_out = 0, s_items = 0, s_items2 = 0;
  for (int c = c0; c < min(c0 + per, K); ++c) {
    int64_t n = counts[c];
    int64_t S = seg_off[c + 1] - seg_off[c];
    int64_t T = tile_off[c + 1] - tile_off[c];
    int64_t i1, i2;
    items(n, T, i1, i2);
    s_cnt += n;
    s_out += n * S;
    s_items += i1;
    s_items2 += i2;
  }
  int64_t tot_cnt, tot_out, tot_items, tot_items2;
  int64_t p_cnt = block_exclusive_scan<int64_t>(s_cnt, &tot_cnt, sbuf);
  int64_t p_out = block_exclusive_scan<int64_t>(s_out, &tot_out, sbuf);
  int64_t p_items = block_exclusive_scan<int64_t>(s_items, &tot_items, sbuf);
  int64_t p_items2 = block_exclusive_scan<int64_t>(s_items2, &tot_items2, sbuf);
  for (int c = c0; c < min(c0 + per, K); ++c) {
    int64_t n = counts[c];
    int64_t S = seg_off[c + 1] - seg_off[c];
    int64_t T = tile_off[c + 1] - tile_off[c];
    int64_t i1, i2;
    items(n, T, i1, i2);
    probe_off[c] = static_cast<int32_t>(p_cnt);
    outbase[c] = p_out;
    item_off[c] = p_items;
    if (item_off2) item_off2[c] = p_items2;
    cursor[c] = 0;
    p_cnt += n;
    p_out += n * S;
    p_items += i1;
    p_items2 += i2;
  }
  if (threadIdx.x == 0) {
    probe_off[K] = static_cast<int32_t>(tot_cnt);
    outbase[K] = tot_out;
    item_off[K] = tot_items;
    if (item_off2) item_off2[K] = tot_items2;
    meta[M_ITEMS] = tot_items;
    meta[M_ITEMS2] = tot_items2;
    meta[M_OUT_TOTAL] = tot_out;
    meta[M_OVERFLOW] = tot_out > capacity ? 1 : 0;
    meta[M_WORK] = 0;
    meta[M_WORK2] = 0;
    // M_QLO: zeroed before the plan, set by query_lo_kernel / the probe gather
  }
}

// meta[M_QLO] = 1 when some query value is not exactly an fp16 (its lo plane
// is non-zero): the plan's dense split needs it before the probe gather
__global__ void query_lo_kernel(const float* __restrict__ Q, int64_t n4, int64_t* __restrict__ meta) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  bool lo = false;
  for (; i < n4; i += stride) {
    const float4 v = reinterpret_cast<const float4*>(Q)[i];
    lo |= __half2float(__float2half_rn(v.x)) != v.x || __half2float(__float2half_rn(v.y)) != v.y ||
          __half2float(__float2half_rn(v.z)) != v.z || __half2float(__float2half_rn(v.w)) != v.w;
  }
  if (__syncthreads_or(lo) && threadIdx.x == 0)
    atomicOr(reinterpret_cast<unsigned long long*>(meta + M_QLO), 1ull);
}

__global__ void probe_scatter_kernel(const int32_t* __restrict__ cells, int64_t nprobes,
                                     const int32_t* __restrict__ probe_off,
                                     int32_t* __restrict__ cursor, int32_t* __restrict__ probe_list,
                                     int32_t* __restrict__ probe_rank) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nprobes) return;
  int c = cells[i];
  if (c < 0) return;
  int r = atomicAdd(&cursor[c], 1);
  probe_list[probe_off[c] + r] = static_cast<int32_t>(i);
  probe_rank[i] = r;
}

__global__ void compact_zero_kernel(float* __restrict__ out, const int64_t* __restrict__ meta) {
  if (meta[M_OVERFLOW]) return;
  const int64_t n = meta[M_OUT_TOTAL];
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (; i < n; i += stride) out[i] = 0.f;
}

struct ScanArgs {
  gift_fif_view f;
  const float* Q;
  const float* qn2;
  int ma;
  int mode;
  float inv_sigma2;
  bool vec16;
  const int32_t* counts;
  const int32_t* probe_off;
  const int32_t* probe_list;
  const int64_t* outbase;
  const int64_t* item_off;
  float* out;
  int64_t* meta;
};

template <bool A_HALF>
__global__ void __launch_bounds__(simt::NTHR, 2) fif_scan_kernel(ScanArgs p) {
  extern __shared__ __align__(128) char smem[];
  __shared__ int64_t s_item;
  __shared__ int64_t s_brow[simt::TB];
  __shared__ float s_qn2[simt::TB];
  __shared__ float s_pn2[simt::TA];
  __shared__ int32_t s_sp[simt::TA + 2];
  const int tid = threadIdx.x;
  const gift_fif_view& f = p.f;
  if (p.meta[M_OVERFLOW]) return;
  const int64_t n_items = p.meta[M_ITEMS];
  const int K = f.K, d = f.d;
  for (;;) {
    if (tid == 0) s_item = static_cast<int64_t>(atomicAdd(reinterpret_cast<unsigned long long*>(&p.meta[M_WORK]), 1ull));
    __syncthreads();
    const int64_t item = s_item;
    if (item >= n_items) break;
    // cell = largest c with item_off[c] <= item (item_off non-decreasing)
    int lo = 0, hi = K - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (p.item_off[mid] <= item)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int c = lo;
    const int64_t rem = item - p.item_off[c];
    const int cnt = p.counts[c];
    const int nm = (cnt + simt::TB - 1) / simt::TB;
    const int64_t t = f.tile_off[c] + rem / nm;
    const int mt = static_cast<int>(rem % nm);
    const int p0 = f.tile_pstart[t], p1 = f.tile_pend[t];
    const int seg0 = f.tile_seg0[t], seg1 = f.tile_seg1[t];
    const int nb = min(simt::TB, cnt - mt * simt::TB);
    const int pb0 = p.probe_off[c] + mt * simt::TB;
    if (tid < simt::TB) {
      if (tid < nb) {
        int pr = p.probe_list[pb0 + tid];
        int64_t view = pr / p.ma;
        s_brow[tid] = view;
        s_qn2[tid] = p.qn2[view];
      } else {
        s_brow[tid] = 0;
        s_qn2[tid] = 0.f;
      }
    }
    if (tid < simt::TA) s_pn2[tid] = (p0 + tid < p1) ? f.pnorm2[p0 + tid] : 0.f;
    const int nseg = seg1 - seg0;
    for (int i = tid; i <= nseg; i += simt::NTHR) s_sp[i] = f.seg_pstart[seg0 + i];
    __syncthreads();

    simt::TileRows tr;
    tr.a_base = f.feat;
    tr.b_base = p.Q;
    tr.na = p1 - p0;
    tr.nb = nb;
    tr.d = d;
    float acc[8][4];
    simt::mainloop<A_HALF>(
        smem, tr, [&](int r) -> int64_t { return static_cast<int64_t>(p0) + r; },
        [&](int r) -> int64_t { return s_brow[r]; }, p.vec16, acc);

    // epilogue 1: transformed dot tile -> smem
    float* Ds = reinterpret_cast<float*>(smem);
    const simt::Lanes L;
    const bool gauss = p.mode == GIFT_SIM_GAUSSIAN;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = L.a_row(i);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = L.b_row(j);
        float v = acc[i][j];
        if (gauss) v = 2.0f * v - s_pn2[r];  // max_p(2q.p - |p|^2) <-> min_p |q-p|^2
        Ds[r * simt::DS_STRIDE + m] = v;
      }
    }
    __syncthreads();
    // epilogue 2: max over each segment's rows, similarity, store
    const int64_t S_c = f.seg_off[c + 1] - f.seg_off[c];
    const int64_t seg_base = f.seg_off[c];
    const int64_t obase = p.outbase[c];
    for (int idx = tid; idx < nseg * nb; idx += simt::NTHR) {
      const int m = idx / nseg;
      const int sl = idx - m * nseg;
      const int sp0 = s_sp[sl], sp1 = s_sp[sl + 1];
      const int r0 = max(sp0, p0) - p0, r1 = min(sp1, p1) - p0;
      float mx = -INFINITY;
      for (int r = r0; r < r1; ++r) mx = fmaxf(mx, Ds[r * simt::DS_STRIDE + m]);
      float sim;
      if (gauss)
        sim = expf(-fmaxf(s_qn2[m] - mx, 0.f) * p.inv_sigma2);
      else
        sim = fminf(fmaxf(mx, 0.f), 1.f);
      const int64_t o = obase + static_cast<int64_t>(mt * simt::TB + m) * S_c + (seg0 + sl - seg_base);
      if (sp0 < p0 || sp1 > p1)
        atomicMax(reinterpret_cast<int*>(p.out + o), __float_as_int(sim));
      else
        p.out[o] = sim;
    }
    __syncthreads();
  }
}

struct ProbeRange {
  int32_t sa, sb;  // segment sub-range of the probe's cell inside a shape range
  int64_t base;    // compact index of (probe, segment 0 of the cell)
  int64_t seg0;    // first segment of the cell
};

// One thread per (probe, shape range): the segment sub-range of the probe's
// cell whose shapes fall inside the range (binary searches done in parallel,
// not on the reduce kernel's critical path).
__global__ void probe_ranges_kernel(const int32_t* __restrict__ cells,
                                    const int32_t* __restrict__ probe_rank,
                                    const int64_t* __restrict__ seg_off,
                                    const int32_t* __restrict__ seg_ord,
                                    const int64_t* __restrict__ outbase,
                                    const int64_t* __restrict__ meta, int64_t nprobes,
                                    int n_ranges, int rs, int64_t n_local, int64_t ord_base,
                                    ProbeRange* __restrict__ rng) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nprobes * n_ranges || meta[M_OVERFLOW]) return;
  const int64_t probe = t / n_ranges;
  const int r = static_cast<int>(t - probe * n_ranges);
  const int c = cells[probe];
  ProbeRange pr{0, 0, 0, 0};
  if (c >= 0) {
    const int64_t b0 = seg_off[c], b1 = seg_off[c + 1];
    int64_t l = b0, h = b1;
    if (n_ranges > 1) {
      const int64_t glo = ord_base + static_cast<int64_t>(r) * rs;
      const int64_t ghi = ord_base + min64(static_cast<int64_t>(r + 1) * rs, n_local);
      while (l < h) {
        int64_t mid = (l + h) >> 1;
        if (seg_ord[mid] < glo) l = mid + 1; else h = mid;
      }
      int64_t l2 = l;
      h = b1;
      while (l2 < h) {
        int64_t mid = (l2 + h) >> 1;
        if (seg_ord[mid] < ghi) l2 = mid + 1; else h = mid;
      }
      h = l2;
    }
    pr.sa = static_cast<int32_t>(l - b0);
    pr.sb = static_cast<int32_t>(h - b0);
    pr.base = outbase[c] + static_cast<int64_t>(probe_rank[probe]) * (b1 - b0);
    pr.seg0 = b0;
  }
  rng[t] = pr;
}

struct ReduceArgs {
  const ProbeRange* rng;      // [B*V*ma, n_ranges]
  const int32_t* seg_ord;
  const float* out;
  const int64_t* meta;
  const int32_t* vq;
  int V, ma, n_ranges, rs;
  int64_t n_local, ord_base;
  double* scores;
  int cand_k;        // > 0: also emit the range's best cand_k (score desc, ordinal asc)
  double* cand_s;    // [B][n_ranges][cand_k]
  int32_t* cand_i;   // global ordinals, -1 padded
};

constexpr int RED_MAXK = 8;

// candidate order: score descending, then global ordinal ascending (-1 =
// none sorts last)
__device__ __forceinline__ bool cand_better(double s1, int32_t o1, double s2, int32_t o2) {
  return s1 > s2 || (s1 == s2 && static_cast<uint32_t>(o1) < static_cast<uint32_t>(o2));
}

// Sorted best-ck insertion (score desc, ordinal asc) into per-thread lists.
__device__ __forceinline__ void cand_insert(double (&ls)[RED_MAXK], int32_t (&lo)[RED_MAXK],
                                            int ck, double xs, int32_t xo) {
  double lastv = ls[0];  // ls[ck - 1] without dynamic register indexing
  int32_t lasto = lo[0];
#pragma unroll
  for (int t = 1; t < RED_MAXK; ++t)
    if (t == ck - 1) {
      lastv = ls[t];
      lasto = lo[t];
    }
  if (!cand_better(xs, xo, lastv, lasto)) return;
#pragma unroll
  for (int t = 0; t < RED_MAXK; ++t) {
    if (t < ck && cand_better(xs, xo, ls[t], lo[t])) {
      const double ys = ls[t];
      const int32_t yo = lo[t];
      ls[t] = xs;
      lo[t] = xo;
      xs = ys;
      xo = yo;
    }
  }
}

// Warp: the ck best of the lanes' sorted lists, in order, via ck rounds of
// argmax; lane 0 receives them in (os, oo).
__device__ __forceinline__ void warp_select(double (&ls)[RED_MAXK], int32_t (&lo)[RED_MAXK],
                                            int ck, double* os_out, int32_t* oo_out) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < RED_MAXK; ++r) {
    if (r >= ck) break;
    double bs = ls[0];
    int32_t bo = lo[0];
    int bl = lane;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, off);
      const int32_t oo = __shfl_xor_sync(0xffffffffu, bo, off);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
      if (cand_better(os, oo, bs, bo) || (os == bs && oo == bo && ol < bl)) {
        bs = os;
        bo = oo;
        bl = ol;
      }
    }
    if (lane == 0) {
      os_out[r] = bs;
      oo_out[r] = bo;
    }
    if (lane == bl) {  // pop the winner's head
#pragma unroll
      for (int t = 0; t + 1 < RED_MAXK; ++t) {
        ls[t] = ls[t + 1];
        lo[t] = lo[t + 1];
      }
      ls[RED_MAXK - 1] = -INFINITY;
      lo[RED_MAXK - 1] = -1;
    }
  }
}

// Per (query, shape range of rs shapes): every (view, slot) probe's
// per-segment maxima are max-ed into vb[view][shape] (shared, atomicMax on
// non-negative float bits: order-independent) in one parallel pass; then each
// shape's column is summed in view order in f64 and divided by Vq —
// total += view_best, score = total / Vq (matching.py:153-161), same add order.
__global__ void __launch_bounds__(RED_THREADS) fif_reduce_kernel(ReduceArgs a) {
  extern __shared__ __align__(128) char smem[];
  float* vb = reinterpret_cast<float*>(smem);  // [V][rs]
  if (a.meta[M_OVERFLOW]) return;
  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const int rg = blockIdx.x;
  const int rs = a.rs;
  const int64_t lo = static_cast<int64_t>(rg) * rs;
  const int n = static_cast<int>(min64(lo + rs, a.n_local) - lo);
  const int64_t glo = a.ord_base + lo;
  const int V = a.V;
  for (int i = tid; i < (V * rs) >> 2; i += RED_THREADS)
    reinterpret_cast<float4*>(vb)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = ((V * rs) & ~3) + tid; i < V * rs; i += RED_THREADS) vb[i] = 0.f;
  __syncthreads();
  const int64_t pbase = static_cast<int64_t>(b) * V * a.ma;
  const int nslot = V * a.ma;
  // warp w owns slots [w * per, (w + 1) * per)
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int NW = RED_THREADS / 32;
  const int per = (nslot + NW - 1) / NW;
  const int s0 = warp * per, s1 = min(nslot, s0 + per);
  // shapes with a positive view best: the only columns worth summing
  __shared__ uint32_t s_touch[RED_MAX_RS / 32];
  __shared__ int s_list[RED_MAX_RS];
  __shared__ int s_nt;
  for (int i = tid; i < RED_MAX_RS / 32; i += RED_THREADS) s_touch[i] = 0u;
  if (tid == 0) s_nt = 0;
  __syncthreads();
  auto put = [&](int row, int o, float val) {
    atomicMax(reinterpret_cast<int*>(vb + row * rs + o), __float_as_int(val));
    if (val > 0.f) atomicOr(&s_touch[o >> 5], 1u << (o & 31));
  };
  constexpr int RED_UNROLL = 4;
  for (int c0 = s0; c0 < s1; c0 += 32) {
    // lane j holds slot c0 + j's range
    const int sj = c0 + lane;
    ProbeRange pr{0, 0, 0, 0};
    if (sj < s1) pr = a.rng[(pbase + sj) * a.n_ranges + rg];
    const int len = pr.sb - pr.sa;
    const int maxlen = __reduce_max_sync(0xffffffffu, len);
    const int total = __reduce_add_sync(0xffffffffu, len);
    if (maxlen * 32 <= 2 * total + 64) {
      // balanced: every lane walks its own slot, RED_UNROLL items per pass
      // with all loads issued before the first atomic
      const int row = sj / a.ma;
      for (int k0 = 0; k0 < maxlen; k0 += RED_UNROLL) {
        int oo[RED_UNROLL];
        float vv[RED_UNROLL];
#pragma unroll
        for (int u = 0; u < RED_UNROLL; ++u) {
          const int k = pr.sa + k0 + u;
          if (k0 + u < len) {
            oo[u] = static_cast<int>(a.seg_ord[pr.seg0 + k] - glo);
            vv[u] = a.out[pr.base + k];
          }
        }
#pragma unroll
        for (int u = 0; u < RED_UNROLL; ++u)
          if (k0 + u < len) put(row, oo[u], vv[u]);
      }
      continue;
    }
    // skewed: the warp's (slot, segment) pairs are flattened so every lane
    // has work (slot of item `it` found by a shuffle search over the
    // exclusive prefix of the lengths)
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - len;
    for (int it0 = 0; it0 < total; it0 += 32 * RED_UNROLL) {  // warp-uniform trip count
      int oo[RED_UNROLL], row[RED_UNROLL];
      float vv[RED_UNROLL];
#pragma unroll
      for (int u = 0; u < RED_UNROLL; ++u) {
        const int it = it0 + u * 32 + lane;
        int j = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int cand = j + step;
          const int ex = __shfl_sync(0xffffffffu, excl, cand);
          if (cand < 32 && ex <= it) j = cand;
        }
        const int ej = __shfl_sync(0xffffffffu, excl, j);
        const int saj = __shfl_sync(0xffffffffu, pr.sa, j);
        const int64_t seg0 = __shfl_sync(0xffffffffu, pr.seg0, j);
        const int64_t base = __shfl_sync(0xffffffffu, pr.base, j);
        row[u] = -1;
        if (it < total) {
          const int k = saj + (it - ej);
          oo[u] = static_cast<int>(a.seg_ord[seg0 + k] - glo);
          vv[u] = a.out[base + k];
          row[u] = (c0 + j) / a.ma;
        }
      }
#pragma unroll
      for (int u = 0; u < RED_UNROLL; ++u)
        if (row[u] >= 0) put(row[u], oo[u], vv[u]);
    }
  }
  __syncthreads();
  // touched shapes -> list; each one's column is summed in view order in f64
  // (untouched columns are all zero: their sum is exactly 0.0) and the f64
  // total parked in rows 0-1 of its own column
  for (int o = tid; o < n; o += RED_THREADS)
    if ((s_touch[o >> 5] >> (o & 31)) & 1u) s_list[atomicAdd(&s_nt, 1)] = o;
  __syncthreads();
  const int nt = s_nt;
  for (int t = tid; t < nt; t += RED_THREADS) {
    const int o = s_list[t];
    double acc = 0.0;
    for (int v = 0; v < V; ++v) acc += static_cast<double>(vb[v * rs + o]);
    const int2 w = make_int2(__double2loint(acc), __double2hiint(acc));
    vb[o] = __int_as_float(w.x);
    vb[rs + o] = __int_as_float(w.y);
  }
  __syncthreads();
  const double denom = static_cast<double>(a.vq ? a.vq[b] : V);
  const int ck = a.cand_k;
  double ls[RED_MAXK];
  int32_t lo_[RED_MAXK];
#pragma unroll
  for (int i = 0; i < RED_MAXK; ++i) {
    ls[i] = -INFINITY;
    lo_[i] = -1;
  }
  for (int o = tid; o < n; o += RED_THREADS) {
    const bool hit = (s_touch[o >> 5] >> (o & 31)) & 1u;
    const double acc =
        hit ? __hiloint2double(__float_as_int(vb[rs + o]), __float_as_int(vb[o])) : 0.0;
    const double sc = acc / denom;
    if (a.scores) a.scores[static_cast<int64_t>(b) * a.n_local + lo + o] = sc;
    if (ck > 0) cand_insert(ls, lo_, ck, sc, static_cast<int32_t>(glo + o));
  }
  if (ck > 0) {
    // per warp: ck rounds of argmax over the lanes' lists; then warp 0 over
    // the warps' lists
    __shared__ double s_bs[NW][RED_MAXK];
    __shared__ int32_t s_bo[NW][RED_MAXK];
    double os[RED_MAXK];
    int32_t oo[RED_MAXK];
    warp_select(ls, lo_, ck, os, oo);
    if (lane == 0)
#pragma unroll
      for (int r = 0; r < RED_MAXK; ++r) {
        s_bs[warp][r] = r < ck ? os[r] : -INFINITY;
        s_bo[warp][r] = r < ck ? oo[r] : -1;
      }
    __syncthreads();
    if (tid < 32) {
#pragma unroll
      for (int r = 0; r < RED_MAXK; ++r) {
        ls[r] = lane < NW ? s_bs[lane][r] : -INFINITY;
        lo_[r] = lane < NW ? s_bo[lane][r] : -1;
      }
      warp_select(ls, lo_, ck, os, oo);
      if (lane == 0) {
        const int64_t at = (static_cast<int64_t>(b) * a.n_ranges + rg) * ck;
#pragma unroll
        for (int r = 0; r < RED_MAXK; ++r)
          if (r < ck) {
            a.cand_s[at + r] = oo[r] >= 0 ? os[r] : 0.0;
            a.cand_i[at + r] = oo[r];
          }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Shape-centric gather reduce (indexes carrying the shape -> segment map).
//
// The per-range reduce above zeroes and sums a [V x rs] view-best tile per
// (query, shape range): B * N * V shared-memory work per batch, which at 1M
// shapes dwarfs the compact buffer itself.  Here every (query, shape) pair is
// visited once instead.  A CTA owns G queries x rs shapes; it first folds its
// queries' probes into shared tables: a bitmap over the K cells (cell probed
// by the query?) with per-word prefix counts, and for each probed cell the
// bit set of query slots (slot j = view * ma + ma-slot) that probed it.  A
// thread then takes one shape, tests the cells of its segments against the
// bitmap, ORs the slot sets of the hits and walks the set bits in ascending
// order: bit j names exactly one probe (cell c_j, row base_j of the compact
// buffer) and the shape's segment g in c_j, whose best similarity is
// compact[base_j + g].  The ma slots of a view are max-ed and views are summed
// in ascending view order in f64 (the reference's `total += view_best`
// order, matching.py:153-161): scores are deterministic and bit-identical to
// the per-range reduce; untouched shapes stay exactly 0.  Scores are staged
// in shared memory and one warp per query selects the range's best cand_k.
constexpr int GR_THREADS = 256;
constexpr int GR_G = 4;         // queries per CTA (fewer when the grid would under-fill)
constexpr int GR_SEGC = 4;      // shape segments cached in registers
// probed cells of a shape kept in registers for the slot lookups: 16 with
// many slots (config 3: 0.83 -> 0.65 ms), 8 with one slot word (config 4,
// where 16 spills: 2.1 -> 2.7 ms)
template <int W>
__host__ __device__ constexpr int gr_pc() { return W >= 2 ? 16 : 8; }
constexpr int GR_MAXK = 16384;  // cells covered by the shared-memory bitmap
constexpr int GR_RS_SMALL = 256, GR_RS_LARGE = 1024;

int gather_rs(int64_t n_local) {
  return static_cast<int>(min64(n_local >= 262144 ? GR_RS_LARGE : GR_RS_SMALL, max64(n_local, 1)));
}

// Per (query, slot): the compact offset of the probe's row minus the cell's
// first segment, so that compact[slot_base + global segment] is the probe's
// best similarity for that segment.
__global__ void probe_slot_kernel(const int32_t* __restrict__ cells,
                                  const int32_t* __restrict__ probe_rank,
                                  const int64_t* __restrict__ outbase,
                                  const int64_t* __restrict__ seg_off, int64_t nprobes,
                                  int64_t* __restrict__ slot_base) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nprobes) return;
  const int c = cells[p];
  int64_t v = 0;
  if (c >= 0) {
    const int64_t so = seg_off[c];
    v = outbase[c] + static_cast<int64_t>(probe_rank[p]) * (seg_off[c + 1] - so) - so;
  }
  slot_base[p] = v;
}

struct GatherArgs {
  const int32_t* cells;          // [B * slots] probe cells (-1: zero view)
  const int64_t* slot_base;      // [B * slots]
  const int64_t* shape_seg_off;  // [n_local + 1]
  const int32_t* shape_seg;      // [S] global segment index, ascending cell
  const int32_t* shape_seg_cell; // [S] its cell
  const uint8_t* seg_single;     // [S] the segment's shape has no other segment (or null)
  const int64_t* seg_off;        // [K + 1]
  const int32_t* seg_ord;        // [S] global shape ordinal of each segment
  const float* out;              // compact (probe x segment) best similarities
  const int64_t* meta;
  const int32_t* vq;
  int B, V, ma, K, rs, n_ranges, G;
  int chunk, nchunk;             // owner reduce: segments per item, max items per cell
  int split;                     // owner reduce: single-segment shapes (ma == 1) go to
                                 // fif_owner_fast_kernel (candidate rows in two halves)
  const int64_t* work_off;       // owner reduce: [B * slots + 1] work-list offsets per probe
  int64_t n_local, ord_base;
  double* scores;                // [B][n_local] or null (candidates only)
  int cand_k;
  double* cand_s;                // [B][n_ranges][cand_k]
  int32_t* cand_i;
};

size_t gather_smem(int G, int rs, int K, int slots, int W) {
  const int kw = (K + 31) / 32;
  return static_cast<size_t>(G) * rs * 8           // staged scores
         + static_cast<size_t>(G) * slots * 8      // slot bases
         + static_cast<size_t>(G) * slots * 4      // slot cells
         + static_cast<size_t>(G) * slots * W * 4  // slot sets of the probed cells
         + static_cast<size_t>(G) * kw * 4         // cell bitmap
         + static_cast<size_t>(G) * kw * 2         // prefix counts (u16)
         + static_cast<size_t>(slots) + 16;        // view of each slot (u8)
}

// Shared-memory probe tables of G queries (layout of gather_smem after the
// staged scores).
struct GrTabs {
  int64_t* base;   // [G][slots]
  int32_t* cell;   // [G][slots]
  uint32_t* set;   // [G][slots][W]
  uint32_t* bm;    // [G][kw]
  uint16_t* pre;   // [G][kw]
  uint8_t* view;   // [slots]
  int kw, slots;
};

template <int W>
__device__ __forceinline__ GrTabs carve_tabs(double* after_scores, int G, int slots, int K) {
  GrTabs t;
  t.slots = slots;
  t.kw = (K + 31) >> 5;
  t.base = reinterpret_cast<int64_t*>(after_scores);
  t.cell = reinterpret_cast<int32_t*>(t.base + G * slots);
  t.set = reinterpret_cast<uint32_t*>(t.cell + G * slots);
  t.bm = t.set + G * slots * W;
  t.pre = reinterpret_cast<uint16_t*>(t.bm + G * t.kw);
  t.view = reinterpret_cast<uint8_t*>(t.pre + G * t.kw);
  return t;
}

// Block-wide: fold the probes of queries b0 .. b0+nb-1 into the tables.
template <int W>
__device__ void build_tabs(const GatherArgs& a, const GrTabs& t, int G, int b0, int nb) {
  const int slots = t.slots, kw = t.kw;
  for (int i = threadIdx.x; i < slots; i += blockDim.x) t.view[i] = static_cast<uint8_t>(i / a.ma);
  for (int i = threadIdx.x; i < G * kw; i += blockDim.x) t.bm[i] = 0u;
  for (int i = threadIdx.x; i < G * slots * W; i += blockDim.x) t.set[i] = 0u;
  for (int i = threadIdx.x; i < G * slots; i += blockDim.x) {
    const bool live = i / slots < nb;
    const int64_t p = static_cast<int64_t>(b0) * slots + i;
    t.base[i] = live ? a.slot_base[p] : 0;
    t.cell[i] = live ? a.cells[p] : -1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * slots; i += blockDim.x) {
    const int c = t.cell[i];
    if (c >= 0) atomicOr(t.bm + (i / slots) * kw + (c >> 5), 1u << (c & 31));
  }
  __syncthreads();
  {  // exclusive prefix popcounts of each query's bitmap words (one warp per query)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int g = warp; g < G; g += blockDim.x / 32) {
      int carry = 0;
      for (int w0 = 0; w0 < kw; w0 += 32) {
        const int w = w0 + lane;
        const int c = w < kw ? __popc(t.bm[g * kw + w]) : 0;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (w < kw) t.pre[g * kw + w] = static_cast<uint16_t>(carry + incl - c);
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * slots; i += blockDim.x) {
    const int c = t.cell[i];
    if (c < 0) continue;
    const int g = i / slots, j = i - g * slots;
    const uint32_t word = t.bm[g * kw + (c >> 5)];
    const int rank = t.pre[g * kw + (c >> 5)] + __popc(word & ((1u << (c & 31)) - 1u));
    atomicOr(t.set + (g * slots + rank) * W + (j >> 5), 1u << (j & 31));
  }
  __syncthreads();
}

struct ShapeSegs {
  int64_t g0;
  int nseg;
  int cell[GR_SEGC];
  int32_t seg[GR_SEGC];
};

__device__ __forceinline__ ShapeSegs load_segs(const GatherArgs& a, int64_t s) {
  ShapeSegs h;
  h.g0 = a.shape_seg_off[s];
  h.nseg = static_cast<int>(a.shape_seg_off[s + 1] - h.g0);
#pragma unroll
  for (int j = 0; j < GR_SEGC; ++j) {
    h.seg[j] = j < h.nseg ? a.shape_seg[h.g0 + j] : 0;
    h.cell[j] = j < h.nseg ? a.shape_seg_cell[h.g0 + j] : -1;
  }
  return h;
}

__device__ __forceinline__ bool probed(const GrTabs& t, int g, int c) {
  return (t.bm[g * t.kw + (c >> 5)] >> (c & 31)) & 1u;
}

// f64 sum over the views (ascending) of the best similarity over the view's
// ma slots whose cell holds a segment of the shape: the reference's
// `total += view_best` (matching.py:153-161) for one (query g, shape).
#ifndef OWN_FAST
#define OWN_FAST 4
#endif
#ifndef OWN_CTAS1
#define OWN_CTAS1 4
#endif
template <int W>
__device__ __forceinline__ double pair_acc(const GatherArgs& a, const GrTabs& t, int g,
                                           const ShapeSegs& h) {
  const int kw = t.kw, slots = t.slots;
  const uint32_t* bm = t.bm + g * kw;
  const uint16_t* pre = t.pre + g * kw;
  const uint32_t* set = t.set + g * slots * W;
  uint32_t U[W];
#pragma unroll
  for (int w = 0; w < W; ++w) U[w] = 0u;
  // the shape's probed cells and their segments, kept in registers for the
  // per-bit lookups below (GR_PC of them; more fall back to a global search)
  constexpr int GR_PC = gr_pc<W>();
  int pc[GR_PC];
  int32_t ps[GR_PC];
  int npc = 0;
#pragma unroll
  for (int q = 0; q < GR_PC; ++q) pc[q] = -1;
#pragma unroll
  for (int j = 0; j < GR_SEGC + 1; ++j) {
    // j < GR_SEGC: cached segment j; j == GR_SEGC: the uncached rest
    const int jend = j < GR_SEGC ? min(j + 1, h.nseg) : h.nseg;
    for (int jj = j; jj < jend; ++jj) {
      const int c = j < GR_SEGC ? h.cell[j] : a.shape_seg_cell[h.g0 + jj];
      const uint32_t word = bm[c >> 5];
      if ((word >> (c & 31)) & 1u) {
        const int rank = pre[c >> 5] + __popc(word & ((1u << (c & 31)) - 1u));
#pragma unroll
        for (int w = 0; w < W; ++w) U[w] |= set[rank * W + w];
        const int32_t sgv = j < GR_SEGC ? h.seg[j] : a.shape_seg[h.g0 + jj];
#pragma unroll
        for (int q = 0; q < GR_PC; ++q)
          if (q == npc) {
            pc[q] = c;
            ps[q] = sgv;
          }
        ++npc;
      }
    }
  }
  const int64_t* sb = t.base + g * slots;
  const int32_t* scl = t.cell + g * slots;
  double acc = 0.0;
  float best = 0.f;
  int cur_v = -1;
  // set bits in ascending order, four at a time: the four compact loads are
  // independent (memory-level parallelism), the view fold is serial.
  // Fast path: ma == 1 and a single segment (every bit is its own view in the
  // shape's only cell) -> acc += compact[base_j + seg], j ascending.
  if (a.ma == 1 && h.nseg == 1) {
    // OWN_FAST independent loads per round (config 4: the 20 views of a
    // query probing one cell; the reduce is bound by load latency)
    const int32_t sg0 = h.seg[0];
    while (true) {
      int jj[OWN_FAST];
      bool ok[OWN_FAST];
      float val[OWN_FAST];
#pragma unroll
      for (int q = 0; q < OWN_FAST; ++q) {
        ok[q] = false;
        jj[q] = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          if (!ok[q] && U[w]) {
            jj[q] = w * 32 + (__ffs(U[w]) - 1);
            U[w] &= U[w] - 1u;
            ok[q] = true;
          }
        }
      }
      if (!ok[0]) break;
#pragma unroll
      for (int q = 0; q < OWN_FAST; ++q) val[q] = ok[q] ? a.out[sb[jj[q]] + sg0] : 0.f;
#pragma unroll
      for (int q = 0; q < OWN_FAST; ++q)
        if (ok[q]) acc += static_cast<double>(val[q]);
      if (!ok[OWN_FAST - 1]) break;
    }
  }
  while (true) {
    int jj[4];
    bool ok[4];
    float val[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ok[q] = false;
      jj[q] = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (!ok[q] && U[w]) {
          jj[q] = w * 32 + (__ffs(U[w]) - 1);
          U[w] &= U[w] - 1u;
          ok[q] = true;
        }
      }
    }
    if (!ok[0]) break;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      val[q] = 0.f;
      if (ok[q]) {
        const int cj = scl[jj[q]];
        int32_t sg = -1;
#pragma unroll
        for (int r = 0; r < GR_PC; ++r)
          if (pc[r] == cj) sg = ps[r];
        if (sg < 0 && npc > GR_PC) {  // more probed cells than registers: search
#pragma unroll
          for (int r = 0; r < GR_SEGC; ++r)
            if (h.cell[r] == cj) sg = h.seg[r];
          for (int r = GR_SEGC; sg < 0 && r < h.nseg; ++r)
            if (a.shape_seg_cell[h.g0 + r] == cj) sg = a.shape_seg[h.g0 + r];
        }
        val[q] = a.out[sb[jj[q]] + sg];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (ok[q]) {
        const int v = t.view[jj[q]];
        if (v != cur_v) {  // views ascend with j: flush the previous view's best
          acc += static_cast<double>(best);
          best = 0.f;
          cur_v = v;
        }
        best = fmaxf(best, val[q]);
      }
    }
    if (!ok[3]) break;
  }
  return acc + static_cast<double>(best);
}


template <int W>
__global__ void __launch_bounds__(GR_THREADS) fif_gather_reduce_kernel(GatherArgs a) {
  extern __shared__ __align__(16) double s_sc[];  // [G][rs], then the probe tables
  if (a.meta[M_OVERFLOW]) return;
  const int rg = blockIdx.x;
  const int G = a.G;
  const int b0 = blockIdx.y * G;
  const int nb = min(G, a.B - b0);
  const int64_t lo = static_cast<int64_t>(rg) * a.rs;
  const int n = static_cast<int>(min64(lo + a.rs, a.n_local) - lo);
  const GrTabs t = carve_tabs<W>(s_sc + G * a.rs, G, a.V * a.ma, a.K);
  build_tabs<W>(a, t, G, b0, nb);
  // ---- one thread per shape, G queries each
  for (int i = threadIdx.x; i < n; i += GR_THREADS) {
    const int64_t s = lo + i;
    const ShapeSegs h = load_segs(a, s);
    for (int g = 0; g < nb; ++g) {
      const int b = b0 + g;
      const double acc = pair_acc<W>(a, t, g, h);
      const double denom = static_cast<double>(a.vq ? a.vq[b] : a.V);
      const double score = acc == 0.0 ? 0.0 : acc / denom;
      if (a.scores) a.scores[static_cast<int64_t>(b) * a.n_local + s] = score;
      s_sc[g * a.rs + i] = score;
    }
  }
  if (a.cand_k <= 0) return;
  __syncthreads();
  // one warp per query: lanes keep a sorted best-cand_k of a strided slice
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= nb) return;
  const int g = warp, b = b0 + g;
  const int ck = a.cand_k;
  double ls[RED_MAXK];
  int32_t lo_[RED_MAXK];
#pragma unroll
  for (int q = 0; q < RED_MAXK; ++q) {
    ls[q] = -INFINITY;
    lo_[q] = -1;
  }
  for (int i = lane; i < n; i += 32)  // ordinals ascend within a lane
    cand_insert(ls, lo_, ck, s_sc[g * a.rs + i], static_cast<int32_t>(a.ord_base + lo + i));
  double os[RED_MAXK];
  int32_t oo[RED_MAXK];
  warp_select(ls, lo_, ck, os, oo);
  if (lane == 0) {
    const int64_t at = (static_cast<int64_t>(b) * a.n_ranges + rg) * ck;
#pragma unroll
    for (int r = 0; r < RED_MAXK; ++r)
      if (r < ck) {
        a.cand_s[at + r] = oo[r] >= 0 ? os[r] : 0.0;
        a.cand_i[at + r] = oo[r];
      }
  }
}

// Owner reduce: only the shapes a query touches.  CTA (query b, slot j,
// chunk) serves the chunk-th run of `chunk` segments of cell c_j when j is the
// query's first slot probing c_j; a thread takes one segment's shape and
// scores it only if c_j is the first (lowest) of the shape's cells the query
// probed (its owner), so every touched pair is scored exactly once, with the
// gather reduce's per-pair sum.  Dense scores (if requested) are zeroed
// beforehand; candidates: the CTA's best cand_k, rows [b][slots * nchunk].
// Owner work list: probe p = (query b, slot j) contributes ceil(S_c / chunk)
// work items when j is the query's first slot probing its cell c (else 0).
__global__ void owner_count_kernel(const int32_t* __restrict__ cells,
                                   const int64_t* __restrict__ seg_off, int64_t nprobes, int slots,
                                   int chunk, const int64_t* __restrict__ meta,
                                   int32_t* __restrict__ cnt) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nprobes) return;
  const int c = cells[p];
  int n = 0;
  if (c >= 0 && !meta[M_OVERFLOW]) {
    const int64_t b0 = p - p % slots;
    bool first = true;
    for (int64_t q = b0; q < p; ++q) first &= cells[q] != c;
    if (first) n = static_cast<int>((seg_off[c + 1] - seg_off[c] + chunk - 1) / chunk);
  }
  cnt[p] = n;
}

// candidate lists per owner work item: one per warp (no CTA barrier per item;
// the top-k2 merge downstream takes OWN_WARPS times more candidates)
constexpr int OWN_WARPS = GR_THREADS / 32;

// The probe of work item w: the largest p with work_off[p] <= w, given the
// answer `from` for an earlier item (a few steps forward, else a binary
// search over the rest) -- a CTA's items ascend.
__device__ __forceinline__ int64_t work_probe(const int64_t* __restrict__ work_off,
                                              int64_t nprobes, int64_t w, int64_t from) {
#pragma unroll 1
  for (int step = 0; step < 4; ++step) {
    if (from + 1 >= nprobes || work_off[from + 1] > w) return from;
    ++from;
  }
  int64_t lo = from, hi = nprobes - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (work_off[mid] <= w) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Latency-bound (dependent gathers per pair): 4 CTAs per SM with one slot
// word (64 registers, some spills; config 4: 3.3 -> 2.1 ms per batch), 3 with
// more (80 registers for the larger probed-cell cache; config 3: 0.69 ->
// 0.59 ms).
template <int W>
__global__ void __launch_bounds__(GR_THREADS, W >= 2 ? 3 : OWN_CTAS1) fif_owner_reduce_kernel(GatherArgs a) {
  extern __shared__ __align__(16) double s_tab[];
  if (a.meta[M_OVERFLOW]) return;
  const int slots = a.V * a.ma;
  const int64_t nprobes = static_cast<int64_t>(a.B) * slots;
  const int64_t n_work = a.work_off[nprobes];
  const int ck = a.cand_k;
  const GrTabs t = carve_tabs<W>(s_tab, 1, slots, a.K);
  int tab_b = -1;  // query whose tables are in shared memory
  // contiguous runs of the (query-major) work list per CTA: consecutive items
  // mostly share the query, so its tables are built once per run
  const int64_t per = (n_work + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t w1 = min64(n_work, w0 + per);
  int64_t pr = 0;
  for (int64_t w = w0; w < w1; ++w) {
  // probe of work item w: largest p with work_off[p] <= w (items ascend, so
  // it is at or after the previous item's)
  pr = work_probe(a.work_off, nprobes, w, pr);
  const int b = static_cast<int>(pr / slots), j = static_cast<int>(pr - static_cast<int64_t>(b) * slots);
  const int chunk_id = static_cast<int>(w - a.work_off[pr]);
  const int64_t cand_at =
      ((((static_cast<int64_t>(b) * slots + j) * a.nchunk + chunk_id) * (a.split ? 2 : 1)) *
           OWN_WARPS + (threadIdx.x >> 5)) * static_cast<int64_t>(ck);
  const int c = a.cells[pr];
  const int64_t S_c = a.seg_off[c + 1] - a.seg_off[c];
  const int64_t k0 = static_cast<int64_t>(chunk_id) * a.chunk;
  const int64_t k1 = min64(S_c, k0 + a.chunk);
  if (b != tab_b) {
    __syncthreads();  // previous item's readers are done with the tables
    build_tabs<W>(a, t, 1, b, 1);
    tab_b = b;
  }
  const double denom = static_cast<double>(a.vq ? a.vq[b] : a.V);
  double ls[RED_MAXK];
  int32_t lo_[RED_MAXK];
#pragma unroll
  for (int q = 0; q < RED_MAXK; ++q) {
    ls[q] = -INFINITY;
    lo_[q] = -1;
  }
  const int64_t so = a.seg_off[c];
  for (int64_t k = k0 + threadIdx.x; k < k1; k += GR_THREADS) {
    if (a.split && a.seg_single[so + k]) continue;  // fif_owner_fast_kernel's
    const int32_t ord = a.seg_ord[so + k];
    const int64_t s = ord - a.ord_base;
    ShapeSegs h;
    if (a.seg_single != nullptr && a.seg_single[so + k]) {
      // the shape's only segment is this one (coalesced flag, no lookups)
      h.g0 = 0;
      h.nseg = 1;
#pragma unroll
      for (int r = 0; r < GR_SEGC; ++r) {
        h.seg[r] = r == 0 ? static_cast<int32_t>(so + k) : 0;
        h.cell[r] = r == 0 ? c : -1;
      }
    } else {
      h = load_segs(a, s);
    }
    // owner test: the first of the shape's cells (ascending) the query probed
    int first = -1;
#pragma unroll
    for (int r = 0; r < GR_SEGC; ++r)
      if (first < 0 && r < h.nseg && probed(t, 0, h.cell[r])) first = h.cell[r];
    for (int r = GR_SEGC; first < 0 && r < h.nseg; ++r) {
      const int cc = a.shape_seg_cell[h.g0 + r];
      if (probed(t, 0, cc)) first = cc;
    }
    if (first != c) continue;
    const double acc = pair_acc<W>(a, t, 0, h);
    const double score = acc == 0.0 ? 0.0 : acc / denom;
    if (a.scores) a.scores[static_cast<int64_t>(b) * a.n_local + s] = score;
    if (ck > 0) cand_insert(ls, lo_, ck, score, ord);
  }
  if (ck > 0) {  // this warp's best ck
    double os[RED_MAXK];
    int32_t oo[RED_MAXK];
    warp_select(ls, lo_, ck, os, oo);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int r = 0; r < RED_MAXK; ++r)
        if (r < ck) {
          a.cand_s[cand_at + r] = oo[r] >= 0 ? os[r] : 0.0;
          a.cand_i[cand_at + r] = oo[r];
        }
  }
  }
}

// The owner reduce's single-segment shapes when ma == 1 (config 4: every
// shape's views share one cell): a shape's score is the f64 sum, in slot
// order, of its column over the compact rows of the query's slots probing
// the item's cell -- pair_acc's fast path, the same additions in the same
// order -- with that row list built once per work item instead of per shape,
// in a kernel light enough to keep its candidate lists in registers (the
// general kernel spills them).  Same work list; candidates in the second
// half of each item's candidate row.
__global__ void __launch_bounds__(GR_THREADS) fif_owner_fast_kernel(GatherArgs a) {
  __shared__ int64_t s_ul[128];
  __shared__ int s_nu;
  if (a.meta[M_OVERFLOW]) return;
  const int slots = a.V;  // ma == 1
  const int64_t nprobes = static_cast<int64_t>(a.B) * slots;
  const int64_t n_work = a.work_off[nprobes];
  const int ck = a.cand_k;
  const int lane = threadIdx.x & 31;
  const int64_t per = (n_work + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t w1 = min64(n_work, w0 + per);
  int64_t pr = 0;
  for (int64_t w = w0; w < w1; ++w) {
    pr = work_probe(a.work_off, nprobes, w, pr);  // probe of work item w
    const int b = static_cast<int>(pr / slots), j = static_cast<int>(pr - static_cast<int64_t>(b) * slots);
    const int chunk_id = static_cast<int>(w - a.work_off[pr]);
    const int c = a.cells[pr];
    __syncthreads();  // the previous item's readers of s_ul are done
    if (threadIdx.x < 32) {  // the query's slots probing c, ascending
      int nu = 0;
      const int64_t q0 = static_cast<int64_t>(b) * slots;
      for (int j0 = 0; j0 < slots; j0 += 32) {
        const int jj = j0 + lane;
        const bool hit = jj < slots && a.cells[q0 + jj] == c;
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (hit) s_ul[nu + __popc(bal & ((1u << lane) - 1u))] = a.slot_base[q0 + jj];
        nu += __popc(bal);
      }
      if (lane == 0) s_nu = nu;
    }
    __syncthreads();
    const int nu = s_nu;
    const int64_t so = a.seg_off[c];
    const int64_t S_c = a.seg_off[c + 1] - so;
    const int64_t k0 = static_cast<int64_t>(chunk_id) * a.chunk;
    const int64_t k1 = min64(S_c, k0 + a.chunk);
    const double denom = static_cast<double>(a.vq ? a.vq[b] : a.V);
    double ls[RED_MAXK];
    int32_t lo_[RED_MAXK];
#pragma unroll
    for (int q = 0; q < RED_MAXK; ++q) {
      ls[q] = -INFINITY;
      lo_[q] = -1;
    }
    for (int64_t k = k0 + threadIdx.x; k < k1; k += GR_THREADS) {
      if (!a.seg_single[so + k]) continue;  // the general kernel's
      const int64_t sg = so + k;
      double acc = 0.0;
      int u = 0;
      for (; u + 4 <= nu; u += 4) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = a.out[s_ul[u + q] + sg];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc += static_cast<double>(v[q]);
      }
      for (; u < nu; ++u) acc += static_cast<double>(a.out[s_ul[u] + sg]);
      const int32_t ord = a.seg_ord[sg];
      const double score = acc == 0.0 ? 0.0 : acc / denom;
      if (a.scores) a.scores[static_cast<int64_t>(b) * a.n_local + (ord - a.ord_base)] = score;
      if (ck > 0) cand_insert(ls, lo_, ck, score, ord);
    }
    if (ck > 0) {  // this warp's best ck, second half of the item's row
      double os[RED_MAXK];
      int32_t oo[RED_MAXK];
      warp_select(ls, lo_, ck, os, oo);
      const int64_t at =
          ((((static_cast<int64_t>(b) * slots + j) * a.nchunk + chunk_id) * 2 + 1) * OWN_WARPS +
           (threadIdx.x >> 5)) * static_cast<int64_t>(ck);
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < RED_MAXK; ++r)
          if (r < ck) {
            a.cand_s[at + r] = oo[r] >= 0 ? os[r] : 0.0;
            a.cand_i[at + r] = oo[r];
          }
    }
  }
}

}  // namespace gift

using namespace gift;

#ifdef GIFT_SCAN_EXPERIMENT
namespace gift {
extern int g_scan_experiment;
extern unsigned long long* g_scan_trace;
}
#endif

namespace {
struct ScoreWs {
  int64_t* meta;
  uint8_t* nz;
  float* qn2;
  int32_t* cells;
  int32_t* counts;
  int32_t* cursor;
  int32_t* probe_off;
  int64_t* outbase;
  int64_t* item_off;
  int64_t* item_off2;
  int32_t* probe_list;
  int32_t* probe_rank;
  void* qws;
  size_t qws_bytes;
  float* compact;
  int64_t capacity;
  __half* g1;
  __half* g2;
  float* qn2s;
  ProbeRange* rng;
  int64_t* slot_base;  // gather reduce: [B * V * ma]
  int32_t* own_cnt;    // owner reduce: work items per probe
  int64_t* own_off;    // [nprobes + 1]
  void* own_ws;        // scan workspace
  size_t own_ws_bytes;
};

bool use_tc(const gift_fif_view* f) {
  if (f->flags & GIFT_FIF_SCAN_SIMT) return false;  // the CUDA-core scan, by request
  return tc_supported(f);
}

int reduce_rs(int64_t V, int64_t n_local) {
  int rs = static_cast<int>(RED_SMEM / (4 * max64(V, 1)));
  rs = max(32, min(rs, RED_MAX_RS)) / 32 * 32;
  return static_cast<int>(max64(min64(rs, n_local), 1));
}

constexpr int OWN_CHUNK = 4096;  // owner reduce: segments per CTA

enum ReduceMode { RM_RANGE = 0, RM_GATHER = 1, RM_OWNER = 2 };

// Mask words of the gather / owner reduce (0: not applicable -> per-range).
int gather_words(const gift_fif_view* f, int V, int ma) {
  if (f->shape_seg_off == nullptr || f->shape_seg == nullptr || f->shape_seg_cell == nullptr)
    return 0;
  const int64_t slots = static_cast<int64_t>(V) * ma;
  if (slots > 128 || f->K > GR_MAXK) return 0;
  return slots <= 32 ? 1 : slots <= 64 ? 2 : 4;
}

// GIFT_FIF_REDUCE(m) in the view flags forces one reduce.  Default: the owner
// reduce (touched pairs only) on large shards, whose per-range [V x rs]
// tiles cost B * N * V: measured 4.1 vs 28 ms on config 4 (1M shapes),
// 1.2 vs 3.1 ms on config 3 (100k); the per-range reduce on small shards
// (config 2, 10k shapes: 0.10 vs 0.37 ms).
constexpr int64_t OWNER_MIN_SHAPES = 32768;

int reduce_mode(const gift_fif_view* f, int V, int ma) {
  const int W = gather_words(f, V, ma);
  if (W == 0) return RM_RANGE;
  switch ((f->flags >> GIFT_FIF_REDUCE_SHIFT) & 3) {
    case GIFT_FIF_REDUCE_RANGE: return RM_RANGE;
    case GIFT_FIF_REDUCE_GATHER: return RM_GATHER;
    case GIFT_FIF_REDUCE_OWNER: return RM_OWNER;
    default: break;
  }
  return f->n_local >= OWNER_MIN_SHAPES ? RM_OWNER : RM_RANGE;
}

// single-segment shapes of an ma == 1 query batch on fif_owner_fast_kernel
bool owner_split(const gift_fif_view* f, int V, int ma) {
  return ma == 1 && f->seg_single != nullptr && V <= 128;
}

int owner_nchunk(const gift_fif_view* f) {
  return static_cast<int>(max64(1, cdiv(max64(f->max_cell_segments, 1), OWN_CHUNK)));
}

bool carve(Arena& ar, const gift_fif_view* f, int64_t nviews, int V, int ma, ScoreWs& w) {
  const int K = f->K;
  const int64_t nprobes = nviews * ma;
  w.meta = ar.take<int64_t>(8);
  w.nz = ar.take<uint8_t>(nviews);
  w.qn2 = ar.take<float>(nviews);
  w.cells = ar.take<int32_t>(nprobes);
  w.counts = ar.take<int32_t>(K);
  w.cursor = ar.take<int32_t>(K);
  w.probe_off = ar.take<int32_t>(K + 1);
  w.outbase = ar.take<int64_t>(K + 1);
  w.item_off = ar.take<int64_t>(K + 1);
  w.item_off2 = ar.take<int64_t>(K + 1);
  w.probe_list = ar.take<int32_t>(nprobes);
  w.probe_rank = ar.take<int32_t>(nprobes);
  w.qws_bytes = gift_quantize_ws_bytes(nviews, f->d, K, GIFT_F32);
  w.qws = ar.take<char>(static_cast<int64_t>(w.qws_bytes));
  w.rng = nullptr;
  w.slot_base = nullptr;
  w.own_cnt = nullptr;
  w.own_off = nullptr;
  w.own_ws = nullptr;
  w.own_ws_bytes = 0;
  if (reduce_mode(f, V, ma) != RM_RANGE) {
    w.slot_base = ar.take<int64_t>(nprobes);
    if (!w.slot_base) return false;
    if (reduce_mode(f, V, ma) == RM_OWNER) {
      w.own_cnt = ar.take<int32_t>(nprobes);
      w.own_off = ar.take<int64_t>(nprobes + 1);
      w.own_ws_bytes = scan_ws_bytes(nprobes + 1);
      w.own_ws = ar.take<char>(static_cast<int64_t>(w.own_ws_bytes));
      if (!w.own_cnt || !w.own_off || !w.own_ws) return false;
    }
  } else {
    w.rng = ar.take<ProbeRange>(nprobes * cdiv(max64(f->n_local, 1), reduce_rs(V, f->n_local)));
    if (!w.rng) return false;
  }
  w.g1 = w.g2 = nullptr;
  w.qn2s = nullptr;
  if (use_tc(f)) {
    w.g1 = ar.take<__half>(nprobes * f->d + 512);
    w.g2 = ar.take<__half>(nprobes * f->d + 512);
    w.qn2s = ar.take<float>(nprobes + 128);
    if (!w.g1 || !w.g2) return false;
  }
  if (!w.meta || !w.nz || !w.qn2 || !w.cells || !w.counts || !w.cursor || !w.probe_off ||
      !w.outbase || !w.item_off || !w.probe_list || !w.probe_rank || !w.qws)
    return false;
  w.capacity = static_cast<int64_t>(ar.remaining() / sizeof(float));
  w.compact = ar.take<float>(w.capacity);
  return w.capacity > 0 && w.compact != nullptr;
}
}  // namespace

extern "C" size_t gift_fif_score_ws_bytes(const gift_fif_view* f, int32_t B, int32_t V, int32_t ma,
                                          int64_t compact_capacity) {
  Arena ar(nullptr, SIZE_MAX / 2);
  ScoreWs w;
  carve(ar, f, static_cast<int64_t>(B) * V, V, ma, w);
  return align_up(ar.used, 256) + static_cast<size_t>(compact_capacity) * sizeof(float) + 512;
}

extern "C" int gift_fif_score(const gift_fif_view* f, const float* Q, int32_t B, int32_t V,
                              const int32_t* vq, int32_t ma, int32_t mode, double sigma,
                              double* out_scores, void* ws, size_t ws_bytes, void* stream) {
  return gift_fif_score_ex(f, Q, B, V, vq, ma, mode, sigma, out_scores, ws, ws_bytes, stream,
                           nullptr, nullptr);
}

extern "C" int gift_fif_score_ranges(const gift_fif_view* f, int32_t V) {
  return static_cast<int>(cdiv(max64(f->n_local, 1), reduce_rs(V, f->n_local)));
}

extern "C" int gift_fif_reduce_mode(const gift_fif_view* f, int32_t V, int32_t ma) {
  return reduce_mode(f, V, ma);
}

extern "C" int gift_fif_score_ranges2(const gift_fif_view* f, int32_t V, int32_t ma) {
  const int mode = reduce_mode(f, V, ma);
  if (mode == RM_GATHER) return static_cast<int>(cdiv(max64(f->n_local, 1), gather_rs(f->n_local)));
  if (mode == RM_OWNER) return V * ma * owner_nchunk(f) * OWN_WARPS * (owner_split(f, V, ma) ? 2 : 1);
  return gift_fif_score_ranges(f, V);
}

extern "C" int gift_fif_score_ex(const gift_fif_view* f, const float* Q, int32_t B, int32_t V,
                                 const int32_t* vq, int32_t ma, int32_t mode, double sigma,
                                 double* out_scores, void* ws, size_t ws_bytes, void* stream,
                                 void* ev_scan_begin, void* ev_scan_end) {
  return gift_fif_score_ex2(f, Q, B, V, vq, ma, mode, sigma, out_scores, ws, ws_bytes, stream,
                            ev_scan_begin, ev_scan_end, 0, nullptr, nullptr);
}

extern "C" int gift_fif_score_ex2(const gift_fif_view* f, const float* Q, int32_t B, int32_t V,
                                  const int32_t* vq, int32_t ma, int32_t mode, double sigma,
                                  double* out_scores, void* ws, size_t ws_bytes, void* stream,
                                  void* ev_scan_begin, void* ev_scan_end, int32_t cand_k,
                                  double* cand_s, int32_t* cand_i) {
  GIFT_REQUIRE(cand_k >= 0 && cand_k <= RED_MAXK, GIFT_ERR_UNSUPPORTED,
               "cand_k = %d > %d", cand_k, RED_MAXK);
  GIFT_REQUIRE(out_scores != nullptr || cand_k > 0, GIFT_ERR_INVALID,
               "out_scores may be NULL only with cand_k > 0");
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE(f != nullptr, GIFT_ERR_INVALID, "null index");
  GIFT_REQUIRE(((f->flags >> GIFT_FIF_DRAIN_SHIFT) & 31) <= 16, GIFT_ERR_INVALID,
               "drain interval %d > 16 k-blocks", (f->flags >> GIFT_FIF_DRAIN_SHIFT) & 31);
  GIFT_REQUIRE(ma >= 1 && ma <= f->K, GIFT_ERR_INVALID, "ma must be in [1, %d]", f->K);
  GIFT_REQUIRE(mode == GIFT_SIM_COSINE || mode == GIFT_SIM_GAUSSIAN, GIFT_ERR_INVALID, "bad mode");
  GIFT_REQUIRE(mode != GIFT_SIM_GAUSSIAN || sigma > 0, GIFT_ERR_INVALID, "sigma must be > 0");
  GIFT_REQUIRE(f->dtype == GIFT_F32 || f->dtype == GIFT_F16, GIFT_ERR_INVALID, "bad storage");
  GIFT_REQUIRE(f->n_postings < (int64_t(1) << 31), GIFT_ERR_UNSUPPORTED, "too many postings");
  GIFT_REQUIRE(f->n_postings == 0 || f->feat != nullptr || use_tc(f), GIFT_ERR_UNSUPPORTED,
               "index keeps no storage copy of its features: only the tcgen05 scan can run");
  if (B <= 0 || f->n_local <= 0) return GIFT_OK;
  GIFT_REQUIRE(V >= 1, GIFT_ERR_EMPTY, "view set is empty");
  const int64_t nviews = static_cast<int64_t>(B) * V;
  const int64_t nprobes = nviews * ma;
  Arena ar(ws, ws_bytes);
  ScoreWs w;
  GIFT_REQUIRE(carve(ar, f, nviews, V, ma, w), GIFT_ERR_CAPACITY, "score workspace too small");
  const int K = f->K, d = f->d;

  int rc = gift_view_prep(Q, GIFT_F32, nviews, d, w.nz, w.qn2, stream);
  if (rc) return rc;
  rc = quantize_impl(Q, GIFT_F32, nviews, d, f->centroids, f->cnorm2, K, f->cmax_norm, ma, w.nz,
                     -1, w.cells, w.qws, w.qws_bytes, stream, false, w.qn2,
                     !(f->flags & GIFT_FIF_QUANT_SIMT));
  if (rc) return rc;
  GIFT_CUDA_TRY(cudaMemsetAsync(w.counts, 0, sizeof(int32_t) * K, st));
  probe_count_kernel<<<static_cast<unsigned>(cdiv(nprobes, 256)), 256, 0, st>>>(w.cells, nprobes,
                                                                               w.counts);
  GIFT_LAUNCH_CHECK();
  GIFT_CUDA_TRY(cudaMemsetAsync(w.meta + M_QLO, 0, sizeof(int64_t), st));
  const bool dense = use_tc(f) && tc_dense_enabled(f);
  if (dense) {
    const int64_t n4 = nviews * d / 4;  // d % 8 == 0 on the tensor-core path
    query_lo_kernel<<<static_cast<unsigned>(min64(max64(cdiv(n4, 256), 1), sm_count() * 8)), 256, 0,
                      st>>>(Q, n4, w.meta);
    GIFT_LAUNCH_CHECK();
  }
  probe_plan_kernel<<<1, PLAN_THREADS, 0, st>>>(w.counts, K, f->seg_off, f->tile_off, w.probe_off,
                                                w.outbase, w.item_off, w.cursor, w.meta, w.capacity,
                                                use_tc(f) ? 128 : simt::TB,
                                                use_tc(f) && tc_pair_enabled(f) ? 2 : 1,
                                                dense ? DENSE_MIN_PROBES : 0, w.item_off2);
  GIFT_LAUNCH_CHECK();
  probe_scatter_kernel<<<static_cast<unsigned>(cdiv(nprobes, 256)), 256, 0, st>>>(
      w.cells, nprobes, w.probe_off, w.cursor, w.probe_list, w.probe_rank);
  GIFT_LAUNCH_CHECK();
  if (!(f->flags & GIFT_FIF_TILED_SEGMENTS) || !use_tc(f)) {  // atomicMax targets need zeros
    compact_zero_kernel<<<sm_count() * 4, 256, 0, st>>>(w.compact, w.meta);
    GIFT_LAUNCH_CHECK();
  }

  if (use_tc(f)) {
    TcArgs ta;
    ta.item_off = w.item_off;
    ta.item_off2 = w.item_off2;
    ta.counts = w.counts;
    ta.probe_off = w.probe_off;
    ta.probe_list = w.probe_list;
    ta.outbase = w.outbase;
    ta.out = w.compact;
    ta.meta = w.meta;
    ta.tile_off = f->tile_off;
    ta.tile_pstart = f->tile_pstart;
    ta.tile_pend = f->tile_pend;
    ta.tile_seg0 = f->tile_seg0;
    ta.tile_seg1 = f->tile_seg1;
    ta.seg_off = f->seg_off;
    ta.seg_pstart = f->seg_pstart;
    ta.pnorm2 = f->pnorm2;
    ta.qn2 = w.qn2;
    ta.qn2s = w.qn2s;
    ta.K = K;
    ta.d = d;
    ta.ma = ma;
    ta.mode = mode;
    ta.inv_sigma2 = mode == GIFT_SIM_GAUSSIAN ? static_cast<float>(1.0 / (sigma * sigma)) : 0.f;
    ta.has_lo = 0;
    // D1 drain interval (k-blocks): short tensor-core accumulation chains
    // hold the 1e-5 contract; default 8 (with the calibrated truncation
    // compensation: max 2.1e-6 on c4s, 0.65e-6 on c2s against the f64
    // oracle, profiles/r02/drain_interval_error_study_calibrated.jsonl)
    const int dkb = (f->flags >> GIFT_FIF_DRAIN_SHIFT) & 31;
    ta.chunk_kb = dkb == 0 ? 8 : dkb;
    ta.dyn = (f->flags & GIFT_FIF_SCHED_STATIC) ? 0 : 1;
#ifdef GIFT_SCAN_EXPERIMENT
    ta.exp = g_scan_experiment;
    ta.trace = g_scan_trace;
#endif
    {  // the truncation compensation of this launch's chunking
      const int nkb = (d + 63) / 64;
      double s1 = 0, s2 = 0;
      for (int kb0 = 0; kb0 < nkb; kb0 += ta.chunk_kb) {
        const double n = 4.0 * min(ta.chunk_kb, nkb - kb0);  // K = 16 steps per 64-wide block
        s1 += n;
        s2 += n * n * tcomp_ratio(n);
      }
      ta.tcomp_scale = (f->flags & GIFT_FIF_RAW_ACCUM) ? 0.f
                                                       : static_cast<float>(TCOMP_PER_STEP * s2 / s1);
    }
    int rc2 = launch_scan_tc(f, Q, nprobes, ta, w.g1, w.g2, st, ev_scan_begin, ev_scan_end);
    if (rc2) return rc2;
  } else {
    ScanArgs sa;
    sa.f = *f;
    sa.Q = Q;
    sa.qn2 = w.qn2;
    sa.ma = ma;
    sa.mode = mode;
    sa.inv_sigma2 = mode == GIFT_SIM_GAUSSIAN ? static_cast<float>(1.0 / (sigma * sigma)) : 0.f;
    const bool a_half = f->dtype == GIFT_F16;
    const bool aligned = reinterpret_cast<uintptr_t>(f->feat) % 16 == 0 &&
                         reinterpret_cast<uintptr_t>(Q) % 16 == 0;
    sa.vec16 = aligned && (a_half ? d % 8 == 0 : d % 4 == 0);
    sa.counts = w.counts;
    sa.probe_off = w.probe_off;
    sa.probe_list = w.probe_list;
    sa.outbase = w.outbase;
    sa.item_off = w.item_off;
    sa.out = w.compact;
    sa.meta = w.meta;
    const int nblk = sm_count() * 2;
    if (ev_scan_begin) GIFT_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(ev_scan_begin), st));
    if (a_half) {
      GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_scan_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         simt::Cfg<true>::SMEM));
      fif_scan_kernel<true><<<nblk, simt::NTHR, simt::Cfg<true>::SMEM, st>>>(sa);
    } else {
      GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_scan_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         simt::Cfg<false>::SMEM));
      fif_scan_kernel<false><<<nblk, simt::NTHR, simt::Cfg<false>::SMEM, st>>>(sa);
    }
    GIFT_LAUNCH_CHECK();
    if (ev_scan_end) GIFT_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(ev_scan_end), st));
  }

  const int rmode = reduce_mode(f, V, ma);
  if (rmode != RM_RANGE) {
    const int W = gather_words(f, V, ma);
    GatherArgs ga;
    ga.cells = w.cells;
    ga.slot_base = w.slot_base;
    ga.shape_seg_off = f->shape_seg_off;
    ga.shape_seg = f->shape_seg;
    ga.shape_seg_cell = f->shape_seg_cell;
    ga.seg_single = f->seg_single;
    ga.seg_off = f->seg_off;
    ga.seg_ord = f->seg_ord;
    ga.out = w.compact;
    ga.meta = w.meta;
    ga.vq = vq;
    ga.B = B;
    ga.V = V;
    ga.ma = ma;
    ga.K = K;
    ga.n_local = f->n_local;
    ga.ord_base = f->ord_base;
    ga.scores = out_scores;
    ga.cand_k = cand_s != nullptr ? cand_k : 0;
    ga.cand_s = cand_s;
    ga.cand_i = cand_i;
    probe_slot_kernel<<<static_cast<unsigned>(cdiv(nprobes, 256)), 256, 0, st>>>(
        w.cells, w.probe_rank, w.outbase, f->seg_off, nprobes, w.slot_base);
    GIFT_LAUNCH_CHECK();
    if (rmode == RM_OWNER) {
      ga.G = 1;
      ga.rs = 0;
      ga.chunk = OWN_CHUNK;
      ga.nchunk = owner_nchunk(f);
      ga.split = owner_split(f, V, ma) ? 1 : 0;
      ga.n_ranges = V * ma * ga.nchunk * OWN_WARPS * (ga.split ? 2 : 1);
      if (out_scores)
        GIFT_CUDA_TRY(cudaMemsetAsync(out_scores, 0, sizeof(double) * B * f->n_local, st));
      if (ga.cand_k > 0) {  // slots without work keep "no candidate"
        const size_t nc = static_cast<size_t>(B) * ga.n_ranges * ga.cand_k;
        GIFT_CUDA_TRY(cudaMemsetAsync(cand_s, 0, sizeof(double) * nc, st));
        GIFT_CUDA_TRY(cudaMemsetAsync(cand_i, 0xff, sizeof(int32_t) * nc, st));
      }
      owner_count_kernel<<<static_cast<unsigned>(cdiv(nprobes, 256)), 256, 0, st>>>(
          w.cells, f->seg_off, nprobes, V * ma, OWN_CHUNK, w.meta, w.own_cnt);
      GIFT_LAUNCH_CHECK();
      rc = scan_exclusive_i32_to_i64(w.own_cnt, w.own_off, nprobes, true, w.own_ws,
                                     w.own_ws_bytes, st);
      if (rc) return rc;
      ga.work_off = w.own_off;
      const int smem = static_cast<int>(gather_smem(1, 0, K, V * ma, W));
      dim3 grid(static_cast<unsigned>(sm_count() * 8));
      if (W == 1) {
        GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_owner_reduce_kernel<1>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        fif_owner_reduce_kernel<1><<<grid, GR_THREADS, smem, st>>>(ga);
      } else if (W == 2) {
        GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_owner_reduce_kernel<2>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        fif_owner_reduce_kernel<2><<<grid, GR_THREADS, smem, st>>>(ga);
      } else {
        GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_owner_reduce_kernel<4>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        fif_owner_reduce_kernel<4><<<grid, GR_THREADS, smem, st>>>(ga);
      }
      GIFT_LAUNCH_CHECK();
      if (ga.split) {
        fif_owner_fast_kernel<<<grid, GR_THREADS, 0, st>>>(ga);
        GIFT_LAUNCH_CHECK();
      }
      return GIFT_OK;
    }
    ga.rs = gather_rs(f->n_local);
    ga.n_ranges = static_cast<int>(cdiv(f->n_local, ga.rs));
    ga.chunk = ga.nchunk = 0;
    ga.split = 0;
    // queries per CTA: GR_G, fewer when that leaves the GPU under-filled
    ga.G = GR_G;
    while (ga.G > 1 && ga.n_ranges * cdiv(B, ga.G) < 8LL * sm_count()) ga.G >>= 1;
    const int smem = static_cast<int>(gather_smem(ga.G, ga.rs, K, V * ma, W));
    dim3 grid(static_cast<unsigned>(ga.n_ranges), static_cast<unsigned>(cdiv(B, ga.G)));
    if (W == 1) {
      GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_gather_reduce_kernel<1>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      fif_gather_reduce_kernel<1><<<grid, GR_THREADS, smem, st>>>(ga);
    } else if (W == 2) {
      GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_gather_reduce_kernel<2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      fif_gather_reduce_kernel<2><<<grid, GR_THREADS, smem, st>>>(ga);
    } else {
      GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_gather_reduce_kernel<4>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      fif_gather_reduce_kernel<4><<<grid, GR_THREADS, smem, st>>>(ga);
    }
    GIFT_LAUNCH_CHECK();
    return GIFT_OK;
  }
  // shape ranges: a [V x rs] f32 view-best tile of <= RED_SMEM bytes per CTA
  const int rs = reduce_rs(V, f->n_local);
  const int n_ranges = static_cast<int>(cdiv(f->n_local, rs));
  probe_ranges_kernel<<<static_cast<unsigned>(cdiv(nprobes * n_ranges, 256)), 256, 0, st>>>(
      w.cells, w.probe_rank, f->seg_off, f->seg_ord, w.outbase, w.meta, nprobes, n_ranges, rs,
      f->n_local, f->ord_base, w.rng);
  GIFT_LAUNCH_CHECK();
  ReduceArgs ra;
  ra.rng = w.rng;
  ra.seg_ord = f->seg_ord;
  ra.out = w.compact;
  ra.meta = w.meta;
  ra.vq = vq;
  ra.V = V;
  ra.ma = ma;
  ra.n_ranges = n_ranges;
  ra.rs = rs;
  ra.n_local = f->n_local;
  ra.ord_base = f->ord_base;
  ra.scores = out_scores;
  ra.cand_k = cand_s != nullptr ? cand_k : 0;
  ra.cand_s = cand_s;
  ra.cand_i = cand_i;
  const int red_smem = max(V, 2) * rs * 4;  // rows 0-1 also park the f64 totals
  GIFT_CUDA_TRY(cudaFuncSetAttribute(fif_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     red_smem));
  dim3 rgrid(static_cast<unsigned>(n_ranges), static_cast<unsigned>(B));
  fif_reduce_kernel<<<rgrid, RED_THREADS, red_smem, st>>>(ra);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_fif_tile_n(void) { return simt::TA; }
