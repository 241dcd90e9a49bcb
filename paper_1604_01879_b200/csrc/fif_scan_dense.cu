// K3 F-IF scan of the dense cells of an fp16-storage index (config 4's Zipf
// head cells): probe-major CTA-pair tiles, tcgen05.mma cta_group::2,
// M = 256 probes x N = 256 postings per k-step.
//
// Why a second scan kernel.  With fp16 storage the scan is tensor-bound and
// ~97% of config 4's flops sit in the ~10 cells probed by >= 192 query views
// per batch.  The posting-major kernel (fif_scan_tc.cu: M = 128 postings x N
// <= 128 probes on one SM) is limited twice there (per-role clock64 trace,
// tools/scan_trace.py): its MMA warp waits on the TMA ring for twice the MMA
// time of an item (128 B of operands per MMA cycle per SM), and its epilogue
// reduces each shape's segment (20 consecutive postings) across threads.
// Here a CTA pair computes 256 probes x 256 postings per k-step: each CTA
// loads 128 probe rows (A) and one 128-posting tile (B), 32 KB per 512 MMA
// cycles (half the bytes per MMA cycle), and each epilogue thread owns one
// probe's row of a posting tile, so the per-segment max is a running fmaxf
// over its registers and one similarity is stored per (probe, segment).
//
// Work items (the plan's second list, item_off2 / meta[M_ITEMS2]): cell c,
// posting tile pair tp (tiles 2 tp, 2 tp + 1 of the cell: D columns
// [0, 128) and [128, 256)), probe tile mt (CTA r: the cell's probes
// [256 mt + 128 r, + 128)); items of one tile pair are consecutive (their
// shared postings hit L2).  Only fp16-exact query batches (meta[M_QLO] == 0)
// and indexes whose segments fit a tile (GIFT_FIF_TILED_SEGMENTS) take it.
//
// Precision: as fif_scan_tc.cu -- fp16 products exact, fp32 tensor-core
// accumulation drained to registers every `chunk_kb` k-blocks (two
// 256-column TMEM chunk buffers per CTA), truncation compensation folded into
// the epilogue's scale.
//
// Roles (384 threads, 1 CTA / SM; registers rebalanced with setmaxnreg):
//   warp 0      TMA producer (both CTAs: own probe rows + own posting tile)
//   warp 1      MMA issuer (leader CTA)
//   warp 2      scheduler (leader fetches items, pushes them to the peer)
//   warp 3      idle (completes the first warpgroup)
//   warps 4-11  epilogue: group g = warps 4 + 4 g .. (posting tile 2 tp + g);
//               warp w reads TMEM lanes 32 (w % 4) .. 32 (w % 4) + 31
#include <cudaTypedefs.h>

#include "fif_scan_tc.cuh"
#include "tc_ptx.cuh"

namespace gift {
namespace dense {

constexpr int MP = 128;                // probes per CTA = TMEM lanes
constexpr int NP = 128;                // postings per tile (one CTA's B half)
constexpr int N = 2 * NP;              // MMA N
constexpr int PROBE_TILE = 2 * MP;     // probes per pair item
constexpr int BK = 64;                 // fp16 per k-block (128-byte rows)
constexpr int A_TILE = MP * BK * 2;    // 16 KB
constexpr int B_TILE = NP * BK * 2;    // 16 KB
constexpr int STAGE = A_TILE + B_TILE; // 32 KB per k-block
constexpr int NST = 6;
constexpr int RING = NST * STAGE;      // 192 KB
constexpr int IRING = 8;               // decoded items in flight
constexpr int THREADS = 384;
constexpr int SMEM = 1024 + RING;
constexpr uint32_t TMEM_COLS = 512;    // two chunk buffers of N columns

struct Item {
  int c;           // cell (-1: stop)
  int pb0;         // this CTA's first probe row (cell-major probe order)
  int rk0;         // its rank within the cell's probes
  int npv;         // valid probes of this CTA (0 .. 128)
  int prow;        // this CTA's posting tile (B rows)
  int p0[2], p1[2], seg0[2], seg1[2];  // the two tiles (p1 == p0: absent)
};

__device__ __forceinline__ Item decode(const TcArgs& p, const int64_t* item_off2, int64_t item,
                                       int& hint, int rank) {
  int lo = hint;
  if (item_off2[lo + 1] <= item) {
    int step = 1, hi = lo + 1;
    while (hi + step < p.K && item_off2[hi + step] <= item) {
      hi += step;
      step <<= 1;
    }
    lo = hi;
    int top = min(hi + step, p.K) - 1;
    while (lo < top) {
      const int mid = (lo + top + 1) >> 1;
      if (item_off2[mid] <= item) lo = mid; else top = mid - 1;
    }
  }
  hint = lo;
  Item I;
  I.c = lo;
  const int64_t rem = item - item_off2[lo];
  const int cnt = p.counts[lo];
  const int nm = (cnt + PROBE_TILE - 1) / PROBE_TILE;
  const int64_t T = p.tile_off[lo + 1] - p.tile_off[lo];
  const int64_t tp = rem / nm;
  const int mt = static_cast<int>(rem % nm);
  I.rk0 = mt * PROBE_TILE + rank * MP;
  I.npv = max(0, min(MP, cnt - I.rk0));
  I.pb0 = p.probe_off[lo] + I.rk0;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const int64_t tt = 2 * tp + g;
    if (tt < T) {
      const int64_t t = p.tile_off[lo] + tt;
      I.p0[g] = p.tile_pstart[t];
      I.p1[g] = p.tile_pend[t];
      I.seg0[g] = p.tile_seg0[t];
      I.seg1[g] = p.tile_seg1[t];
    } else {
      I.p0[g] = I.p1[g] = I.p0[0];
      I.seg0[g] = I.seg1[g] = 0;
    }
  }
  I.prow = I.p0[rank];
  return I;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// predicated shared store (one @P STS, no branch around it)
__device__ __forceinline__ void sts_pred(uint32_t a, float v, uint32_t pred) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.u32 p, %2, 0;\n"
      "@p st.shared.f32 [%0], %1;\n"
      "}\n" ::"r"(a),
      "f"(v), "r"(pred)
      : "memory");
}

// predicated global store (one @P STG, no branch around it)
__device__ __forceinline__ void st_pred(float* o, float v, bool pred) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %2, 0;\n"
      "@p st.global.f32 [%0], %1;\n"
      "}\n" ::"l"(o),
      "f"(v), "r"(static_cast<int>(pred))
      : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    fif_scan_dense_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmP, const TcArgs p,
                          const int64_t* __restrict__ item_off2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(16) float s_pn[2][NP];  // per group: |p|^2 of the tile's postings
  __shared__ uint32_t s_end[2][NP / 32];       // per group: segment-end columns
  __shared__ float s_emit[2][16][MP];          // per thread: segment maxima of 16 columns
  __shared__ Item s_item[IRING];
  __shared__ __align__(8) uint64_t ifull[IRING], iempty[IRING];
  __shared__ __align__(8) int64_t s_next[IRING];
  __shared__ __align__(8) uint64_t xfull[IRING], xempty[IRING];
  __shared__ __align__(8) uint64_t full[NST], empty[NST], tfull[2], tempty[2];
  __shared__ uint32_t tmem_holder;
  uint8_t* ring = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  if (p.meta[M_OVERFLOW]) return;  // uniform over the grid
  const int64_t n_items = p.meta[M_ITEMS2];
  if (n_items == 0) return;
  const int nkb = (p.d + BK - 1) / BK;
  const int chunk_kb = p.chunk_kb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < IRING; ++r) {
      tc::mbar_init(&xfull[r], 1);
      tc::mbar_init(&xempty[r], 1);
      tc::mbar_init(&ifull[r], 1);
      tc::mbar_init(&iempty[r], (leader ? 2 : 1) + 2);  // producer, [MMA,] 2 epilogue groups
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 2 * 8);  // every epilogue warp of both CTAs
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmQ);
    tc::tma_prefetch(&tmP);
  }
  if (warp == 1) tc::tmem_alloc_2sm<TMEM_COLS>(&tmem_holder);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem_base = tmem_holder;

  // registers: the role warpgroup gives up to 56 per thread, the epilogue
  // warpgroups take 224 (128 accumulators per thread)
  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t lbar0 = tc::mapa(&full[0], 0);  // completion on the leader's barriers
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % IRING, iph = (it / IRING) & 1;
      tc::mbar_wait(&ifull[slot], iph);
      const Item I = s_item[slot];
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&iempty[slot]);
      if (I.c < 0) break;
      if (lane == 0) GIFT_TRACE_K(p, 1, it, 1, clock64());
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(&empty[stage], phase ^ 1);
        if (tc::elect_one()) {
          uint8_t* st = ring + stage * STAGE;
          const uint32_t lbar = lbar0 + stage * 8;
          if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * STAGE);
          tc::tma_load_2d_2sm(st, &tmQ, lbar, kb * BK, I.pb0);
          tc::tma_load_2d_2sm(st + A_TILE, &tmP, lbar, kb * BK, I.prow);
        }
        __syncwarp();
        if (++stage == NST) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) GIFT_TRACE_K(p, 1, it, 2, clock64());
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer (leader)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
    if (leader) {
      int stage = 0;
      uint32_t phase = 0, chunk_ctr = 0;
      const uint32_t idesc = tc::idesc_f16_f32(2 * MP, N);
      for (uint32_t it = 0;; ++it) {
        const uint32_t slot = it % IRING, iph = (it / IRING) & 1;
        tc::mbar_wait(&ifull[slot], iph);
        const Item I = s_item[slot];
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&iempty[slot]);
        if (I.c < 0) break;
        if (lane == 0) GIFT_TRACE_K(p, 1, it, 3, clock64());
        for (int kb0 = 0; kb0 < nkb; kb0 += chunk_kb) {
          const uint32_t buf = chunk_ctr & 1, aph = (chunk_ctr >> 1) & 1;
          tc::mbar_wait(&tempty[buf], aph ^ 1);
          tc::tc_fence_after();
          const uint32_t d = tmem_base + buf * N;
          const int kend = min(kb0 + chunk_kb, nkb);
          for (int kb = kb0; kb < kend; ++kb) {
            tc::mbar_wait(&full[stage], phase);
            tc::tc_fence_after();
            if (tc::elect_one()) {
              uint8_t* st = ring + stage * STAGE;
              const uint64_t a = tc::smem_desc_sw128(st);
              const uint64_t b = tc::smem_desc_sw128(st + A_TILE);
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                const uint64_t adv = static_cast<uint64_t>(k * 2);  // 32 B in 16-B units
                tc::mma_f16_2sm(d, a + adv, b + adv, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
              }
              tc::mma_commit_2sm(&empty[stage], 0x3);
            }
            __syncwarp();
            if (++stage == NST) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (tc::elect_one()) tc::mma_commit_2sm(&tfull[buf], 0x3);
          __syncwarp();
          ++chunk_ctr;
        }
        if (lane == 0) GIFT_TRACE_K(p, 1, it, 4, clock64());
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------ scheduler
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
    if (lane == 0) {
      int hint = 0;
      unsigned long long* work =
          reinterpret_cast<unsigned long long*>(const_cast<int64_t*>(p.meta) + M_WORK2);
      const uint32_t peer_next = tc::mapa(&s_next[0], 1);
      const uint32_t peer_full = tc::mapa(&xfull[0], 1);
      const uint32_t lead_empty = tc::mapa(&xempty[0], 0);
      const int64_t first = blockIdx.x / 2, stride = gridDim.x / 2;
      for (uint32_t it = 0;; ++it) {
        const uint32_t slot = it % IRING, iph = (it / IRING) & 1;
        int64_t item;
        if (leader) {
          item = p.dyn ? static_cast<int64_t>(atomicAdd(work, 1ull))
                       : first + static_cast<int64_t>(it) * stride;
          tc::mbar_wait(&xempty[slot], iph ^ 1);
          tc::st_cluster_u64(peer_next + slot * 8, item);
          tc::mbar_arrive_cluster(peer_full + slot * 8);
        } else {
          tc::mbar_wait_cluster(&xfull[slot], iph);
          item = s_next[slot];
          tc::mbar_arrive_cluster(lead_empty + slot * 8);
        }
        Item I;
        if (item < n_items) {
          I = decode(p, item_off2, item, hint, static_cast<int>(rank));
        } else {
          I.c = -1;
        }
        tc::mbar_wait(&iempty[slot], iph ^ 1);
        s_item[slot] = I;
        tc::mbar_arrive(&ifull[slot]);
        GIFT_TRACE_K(p, 1, it, 0, clock64());
        if (item < n_items) {
          GIFT_TRACE_K(p, 1, it, 8, I.npv);
          GIFT_TRACE_K(p, 1, it, 9, I.c);
        }
        if (item >= n_items) break;
      }
    }
  } else if (warp == 3) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
  } else {
    // ------------------------------------------------------ epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n");
    const int et = threadIdx.x - 128;  // 0 .. 255
    const int g = et >> 7;             // posting tile 2 tp + g = D columns [128 g, 128 g + 128)
    const int e = et & 127;
    const int wq = warp & 3;           // TMEM lane quarter
    const int row = 32 * wq + lane;    // probe row of this CTA's tile
    const int bar_tail = 1 + g, bar_item = 3 + g;
    const bool gauss = p.mode == GIFT_SIM_GAUSSIAN;
    const float tc = p.tcomp_scale, K2 = gauss ? 2.0f : 1.0f;
    const uint32_t tempty_lead = tc::mapa(&tempty[0], 0);
    const uint32_t tm_row = tmem_base + (static_cast<uint32_t>(32 * wq) << 16) + g * NP;
    float* pn_s = s_pn[g];
    uint32_t* end_s = s_end[g];
    uint32_t chunk_ctr = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % IRING, sph = (it / IRING) & 1;
      tc::mbar_wait(&ifull[slot], sph);
      const Item I = s_item[slot];
      named_bar(bar_item, 128);
      if (e == 0) tc::mbar_arrive(&iempty[slot]);
      if (I.c < 0) break;
      if (et == 0) GIFT_TRACE_K(p, 1, it, 5, clock64());
      const int p0 = I.p0[g], ncol = I.p1[g] - p0;
      const int seg0 = I.seg0[g], nseg = I.seg1[g] - seg0;
      // tail inputs, loaded now (their latency overlaps the drains)
      const float pn_e = (gauss && e < ncol) ? p.pnorm2[p0 + e] : 0.f;
      const int st_e = (e >= 1 && e < nseg) ? p.seg_pstart[seg0 + e] - p0 : -1;
      const bool pvalid = row < I.npv;
      const float qn = pvalid ? p.qn2s[I.pb0 + row] : 0.f;
      const int64_t seg_base = p.seg_off[I.c];
      const int64_t S_c = p.seg_off[I.c + 1] - seg_base;
      const int64_t obase = p.outbase[I.c];
      if (e < NP / 32) end_s[e] = 0u;
      float acc[NP];
#pragma unroll
      for (int n = 0; n < NP; ++n) acc[n] = 0.f;
      for (int kb0 = 0; kb0 < nkb; kb0 += chunk_kb) {
        const uint32_t buf = chunk_ctr & 1, aph = (chunk_ctr >> 1) & 1;
        tc::mbar_wait(&tfull[buf], aph);
        tc::tc_fence_after();
        const uint32_t base = tm_row + buf * N;
#pragma unroll
        for (int j = 0; j < NP / 16; j += 2) {
          float v1[16], v2[16];
          tc::tmem_ld_x16(base + j * 16, v1);
          tc::tmem_ld_x16(base + (j + 1) * 16, v2);
          tc::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            acc[j * 16 + i] += v1[i];
            acc[(j + 1) * 16 + i] += v2[i];
          }
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster_relaxed(tempty_lead + buf * 8);
        ++chunk_ctr;
      }
      if (et == 0) GIFT_TRACE_K(p, 1, it, 6, clock64());
      if (ncol <= 0 || I.npv == 0) continue;  // absent tile / no probes: nothing to write
      // segment-end columns of the tile (tiled segments: segment 0 starts at
      // column 0, segment e >= 1 at st_e, the last one ends at ncol - 1)
      pn_s[e] = pn_e;
      named_bar(bar_tail, 128);
      if (et == 0) GIFT_TRACE_K(p, 1, it, 10, clock64());
      if (st_e > 0) atomicOr(&end_s[(st_e - 1) >> 5], 1u << ((st_e - 1) & 31));
      if (e == 0) atomicOr(&end_s[(ncol - 1) >> 5], 1u << ((ncol - 1) & 31));
      named_bar(bar_tail, 128);
      uint32_t em[NP / 32];
#pragma unroll
      for (int w = 0; w < NP / 32; ++w) em[w] = end_s[w];
      if (et == 0) GIFT_TRACE_K(p, 1, it, 11, clock64());
      // one probe's row: v = K2 s - |p|^2 (2 q.p - |p|^2 or q.p), running max
      // over each segment's columns, similarity stored at the segment's end
      float* o = p.out + obase + static_cast<int64_t>(I.rk0 + row) * S_c + (seg0 - seg_base);
      // Straight-line code over the row (no branches: branchy per-block code
      // thrashed the instruction cache): v = K2 s - |p|^2, running max m; at
      // a segment end (predicated) m goes to this thread's slot of the emit
      // buffer and restarts.  Every 16 columns a short loop turns the
      // buffered maxima into similarities and stores them.
      float* eb = s_emit[g][0] + row;  // entry j at eb[j * MP]
      const uint32_t eb_s = tc::smem_addr(eb);
      float m = -INFINITY;
#pragma unroll
      for (int h = 0; h < NP / 16; ++h) {
        const uint32_t bits = (em[h >> 1] >> ((h & 1) * 16)) & 0xffffu;
        uint32_t koff = 0;  // emitted entries x MP x 4 bytes
#pragma unroll
        for (int i4 = 0; i4 < 16; i4 += 4) {
          const float4 pv = *reinterpret_cast<const float4*>(pn_s + 16 * h + i4);
          const float pc[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            // the posting-major kernel's arithmetic, operation for operation
            // (scores independent of which kernel a batch's cell ran on)
            m = fmaxf(m, fmaf(K2, fmaf(acc[16 * h + i4 + i], tc, acc[16 * h + i4 + i]), -pc[i]));
            const uint32_t end = (bits >> (i4 + i)) & 1u;
            sts_pred(eb_s + koff, m, end);
            koff += end << 9;  // MP * 4 bytes
            m = end ? -INFINITY : m;
          }
        }
        const int k = static_cast<int>(koff >> 9);
        for (int j = 0; j < k; ++j) {
          const float x = eb[j * MP];
          const float sim =
              gauss ? expf(-fmaxf(qn - x, 0.f) * p.inv_sigma2) : fminf(fmaxf(x, 0.f), 1.f);
          st_pred(o + j, sim, pvalid && !GIFT_EXP(p, 16));
        }
        o += k;
      }
      if (et == 0) GIFT_TRACE_K(p, 1, it, 12, clock64());
      named_bar(bar_tail, 128);  // s_pn / s_end are reused by the next item
      if (et == 0) GIFT_TRACE_K(p, 1, it, 7, clock64());
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
  }
}

}  // namespace dense

cudaError_t launch_scan_dense(int ctas, cudaStream_t st, const CUtensorMap& mQ,
                              const CUtensorMap& mP, const TcArgs& a, const int64_t* item_off2) {
  cudaError_t e = cudaFuncSetAttribute(dense::fif_scan_dense_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, dense::SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(max(2, ctas / 2 * 2)));
  cfg.blockDim = dim3(dense::THREADS);
  cfg.dynamicSmemBytes = dense::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, dense::fif_scan_dense_kernel, mQ, mP, a, item_off2);
}

}  // namespace gift
