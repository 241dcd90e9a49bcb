// K3 F-IF scan on the 5th-generation tensor cores (tcgen05 + TMA + TMEM).
//
// Same work items and outputs as the CUDA-core scan (fif_scan.cu): one item =
// a posting tile (<= 128 postings of one cell, whole segments) x a tile of up
// to 64 of that cell's probes; output = per (probe, segment) best similarity.
//
// Precision (north_star: scores within 1e-5 relative, gaussian amplifies dot
// errors 8x at sigma = 0.5): every fp32 operand x is split into two fp16
// planes x = h1 + 2^-11 h2 (h1 = rn(x), h2 = rn((x - h1) 2^11), 22 significant
// bits); the dot is  D1 + 2^-11 D2,  D1 = sum a1 b1,  D2 = sum (a1 b2 + a2 b1),
// three kind::f16 MMAs per k-step with fp32 accumulation in TMEM.  fp16
// products are exact in fp32 but the tensor-core accumulate is not: D1 is
// drained to registers every `chunk_kb` k-blocks (and summed there in fp32,
// round-to-nearest) so its accumulation chains stay short; D2 carries terms
// 2^11 smaller and is drained once per item.  Database planes are built once
// (gift_split_planes); query planes per batch (gather_split kernel below).
//
// Warp roles (1 CTA / SM, persistent, static round-robin over items):
//   warp 0      TMA producer: A1[/A2] (postings, 128 x 64 fp16, 128B swizzle)
//               and B1/B2 (probes, 64 or 128 x 64) per k-block into a 3-stage
//               (4-stage without the A2 plane) ring;
//   warp 1      MMA issuer: 2-3 tcgen05.mma (M=128, N=64|128, K=16) per k-step
//               into D1 (double-buffered per chunk) and D2 (per item);
//               tcgen05.commit releases smem stages and hands accumulators over;
//   warps 2..5  epilogue: tcgen05.ld drains (row = TMEM lane), fp32 sums,
//               similarity transform, per-segment max over rows, store.
#include <cudaTypedefs.h>

#include "fif_scan_tc.cuh"
#include "tc_ptx.cuh"

namespace gift {


constexpr int TC_M = 128;
constexpr int TC_NMAX = 128;  // probes per item: N = 64 or 128 (per item)
constexpr int TC_BK = 64;     // fp16 per k-block = 128-byte rows
constexpr int A_TILE = TC_M * TC_BK * 2;     // 16 KB
constexpr int B_BOX = 64 * TC_BK * 2;        //  8 KB (one 64-row TMA box)
constexpr int B_TILE = TC_NMAX * TC_BK * 2;  // 16 KB
// ring budget: three single-CTA stages of A1 A2 B1 B2 (see Ring<> below)
constexpr int STAGE_LO = 2 * A_TILE + 2 * B_TILE;
constexpr int RING_BYTES = 3 * STAGE_LO;  // 192 KB
constexpr int EPI_COLS = 32;  // epilogue stages 32 probe columns at a time
constexpr int ITEM_RING = 8;     // decoded work items in flight (scheduler -> roles)
// TMEM: D1 (hi x hi) double-buffered per k-chunk, drained every chunk_kb
// k-blocks (short tensor-core accumulation chains: the fp32 accumulate is
// not exact); D2 (the 2^-11-scaled correction terms) double-buffered per
// item, drained once per item (its accumulation error is 2^-11 smaller)
constexpr uint32_t TMEM_COLS = 512;  // D1[2][128] | D2[2][128]
constexpr float SPLIT_INV = 1.0f / 2048.0f;

struct ItemInfo {
  int c, mt, p0, p1, seg0, seg1, nb, pb0, n;  // n: MMA N of the item (64 | 128)
  int t;      // global scan tile index
  bool live;  // pair mode: this CTA's posting tile exists (else a duplicate, no output)
};

// Cell of an item: items ascend along each role's loop, so the search starts
// at the previous item's cell (`hint`): one load when the item stays in that
// cell, else a galloping then binary search over item_off[hint+1 .. K-1]
// (a plain binary search over K = 4096 cells is 12 dependent global loads).
// Pair mode: an item is (two consecutive posting tiles, one probe tile); CTA
// `rank` of the pair takes tile 2 tp + rank.
template <bool PAIR>
__device__ __forceinline__ ItemInfo decode_item(const TcArgs& p, int64_t item, int& hint,
                                                int rank) {
  int lo = hint;
  if (p.item_off[lo + 1] <= item) {
    int step = 1, hi = lo + 1;  // item_off[hi] <= item
    while (hi + step < p.K && p.item_off[hi + step] <= item) {
      hi += step;
      step <<= 1;
    }
    lo = hi;
    int top = min(hi + step, p.K) - 1;  // item_off[top + 1] > item (or top == K - 1)
    while (lo < top) {
      int mid = (lo + top + 1) >> 1;
      if (p.item_off[mid] <= item) lo = mid; else top = mid - 1;
    }
  }
  hint = lo;
  ItemInfo I;
  I.c = lo;
  const int64_t rem = item - p.item_off[lo];
  const int cnt = p.counts[lo];
  const int nm = (cnt + TC_NMAX - 1) / TC_NMAX;
  const int64_t T = p.tile_off[lo + 1] - p.tile_off[lo];
  int64_t tt;  // tile index within the cell
  if (PAIR) {
    tt = 2 * (rem / nm) + rank;
    I.mt = static_cast<int>(rem % nm);
    I.live = tt < T;
    if (!I.live) tt -= 1;  // odd tile count: the second CTA recomputes the first tile
  } else {  // neighbouring CTAs share a posting tile (A)
    tt = rem / nm;
    I.mt = static_cast<int>(rem % nm);
    I.live = true;
  }
  const int64_t t = p.tile_off[lo] + tt;
  I.t = static_cast<int>(t);
  I.p0 = p.tile_pstart[t];
  I.p1 = p.tile_pend[t];
  I.seg0 = p.tile_seg0[t];
  I.seg1 = p.tile_seg1[t];
  I.nb = min(TC_NMAX, cnt - I.mt * TC_NMAX);
  I.pb0 = p.probe_off[lo] + I.mt * TC_NMAX;
  I.n = I.nb > 64 ? 128 : 64;
  return I;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// Stage layouts.  Single CTA: A1 [A2] B1 B2 (B = N probe rows).  CTA pair
// (cta_group::2, M = 256): each CTA holds its own posting tile's A1 [A2] and
// half of the probe rows of B1 and B2 (N / 2 each); the pair's MMA reads the
// other halves from the peer's smem at the same offsets.
template <bool PAIR>
struct Ring {
  static constexpr int B_PART = PAIR ? B_TILE / 2 : B_TILE;
  static constexpr int LO = 2 * A_TILE + 2 * B_PART;
  static constexpr int NOLO = A_TILE + 2 * B_PART;
  static constexpr int STAGES_LO = RING_BYTES / LO;      // 3 | 4
  static constexpr int STAGES_NOLO = RING_BYTES / NOLO;  // 4 | 6
};
constexpr int MAX_RING_STAGES = 6;

// Epilogue column groups: the single-CTA kernel (fp16 storage, config 4; its
// epilogue paces the tensor cores) runs two groups of 4 epilogue warps, each
// draining and reducing half of the probe columns; the f32-plane CTA-pair
// kernel (HBM-bound) keeps one group and the shared memory other batches'
// kernels can share an SM with.
template <int G>
struct Epi {
  static constexpr int THREADS = 96 + 128 * G;  // producer, MMA, scheduler, 4 G epilogue
  static constexpr int COLS = G == 1 ? EPI_COLS : EPI_COLS / 2;  // tail slice width
  static constexpr int STRIDE = COLS + 1;
  static constexpr int DS = TC_M * STRIDE;  // floats of one group's staging tile
  static constexpr int SMEM = RING_BYTES + G * DS * 4 + 256;
};

template <bool PAIR, int G, bool LO>
__global__ void __launch_bounds__(Epi<G>::THREADS, 1)
    fif_scan_tc_kernel(const __grid_constant__ CUtensorMap tmA1,
                       const __grid_constant__ CUtensorMap tmA2,
                       const __grid_constant__ CUtensorMap tmB1,
                       const __grid_constant__ CUtensorMap tmB2,
                       const __grid_constant__ CUtensorMap tmB1h,
                       const __grid_constant__ CUtensorMap tmB2h, const TcArgs p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ int32_t s_sp[G * (TC_M + 2)];
  // per epilogue group: the groups run items independently (a group may
  // start the next item's tail while the other finishes this one's), and an
  // item's column split depends on its N
  __shared__ float s_qn2[G * TC_NMAX];
  __shared__ ItemInfo s_item[ITEM_RING];
  __shared__ __align__(8) uint64_t ifull[ITEM_RING], iempty[ITEM_RING];
  // pair: item indices the leader's scheduler fetched, pushed into the peer
  __shared__ __align__(8) int64_t s_next[ITEM_RING];
  __shared__ __align__(8) uint64_t xfull[ITEM_RING], xempty[ITEM_RING];
  float* Ds = reinterpret_cast<float*>(smem + RING_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RING_BYTES + G * Epi<G>::DS * 4);
  uint64_t* full = bars;
  uint64_t* empty = bars + MAX_RING_STAGES;
  uint64_t* tfull = bars + 2 * MAX_RING_STAGES;  // D1 chunk buffers (2, or 4 when qz4)
  uint64_t* tempty = tfull + 4;
  uint64_t* dfull = tempty + 4;                  // D2 item buffers
  uint64_t* dempty = dfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(dempty + 2);
  constexpr bool has_lo = LO;  // the f32 storage's lo plane (compile time: lean MMA loop)
  constexpr int stage_bytes = has_lo ? Ring<PAIR>::LO : Ring<PAIR>::NOLO;
  constexpr int nstages = has_lo ? Ring<PAIR>::STAGES_LO : Ring<PAIR>::STAGES_NOLO;
  constexpr int b_off = has_lo ? 2 * A_TILE : A_TILE;  // B1 offset in a stage
  constexpr int B_PART = Ring<PAIR>::B_PART;
  // combined B operand [b1 | b2] (one N = 2n MMA per k-step, A read once):
  // always on a single CTA; on a pair only without the lo plane (CTA r then
  // holds plane r: the pair's B is exactly [b1 | b2]); a pair with the lo
  // plane keeps three MMAs with half of each plane per CTA and D2 per item
  constexpr bool cb = !PAIR || !has_lo;
  const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  // item sequence: per CTA, or per pair (both CTAs walk the same items)
  const int64_t first = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t stride = PAIR ? gridDim.x / 2 : gridDim.x;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.meta[M_OVERFLOW]) return;  // uniform over the grid (both CTAs of a pair)
  const int64_t n_items = p.meta[M_ITEMS];
  // every query lo plane is zero (fp16-exact queries): the single-CTA kernel
  // drops the b2 operand -- one N = n MMA per k-step instead of N = 2n, no b2
  // loads, no D2 drains (b2 = 0 contributes exactly 0: bit-identical)
  // (pairs without the lo plane too: each CTA then holds half of b1's rows)
  const bool qz = (!PAIR || !LO) && p.meta[M_QLO] == 0;
  // qz without the lo plane needs D1 only (128 TMEM columns per chunk): four
  // chunk buffers instead of two, so the MMAs run a whole item ahead of the
  // epilogue's per-item tail instead of stalling on the accumulators
  const bool qz4 = qz && !LO;
  // a single CTA with fp16-exact queries stages A + b1 only: 32 KB stages, six
  // in the ring instead of four (more k-blocks in flight; measured neutral on
  // config 4, whose scan is paced by its per-item latencies)
  const bool small_st = qz && !PAIR && !LO;
  // ... and two k-blocks per stage (one producer / MMA hand-off per two
  // k-blocks: the per-k-block hand-off paced this scan), when
  // the drain chunks are whole stages
  const int kps = (small_st && p.chunk_kb % 2 == 0) ? 2 : 1;  // k-blocks per stage
  constexpr int SUB = A_TILE + B_TILE;  // one k-block's A + b1 in a small stage
  const int st_bytes = small_st ? kps * SUB : stage_bytes;
  const int n_st = small_st ? RING_BYTES / (kps * SUB) : nstages;
  const uint32_t nbuf = qz4 ? 4u : 2u;
  const uint32_t buf_cols = qz4 ? TC_NMAX : ((!PAIR || !LO) ? 2 * TC_NMAX : TC_NMAX);
  const int nkb = (p.d + TC_BK - 1) / TC_BK;
  const int chunk_kb = p.chunk_kb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < MAX_RING_STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < ITEM_RING; ++r) {
      tc::mbar_init(&xfull[r], 1);
      tc::mbar_init(&xempty[r], 1);
      tc::mbar_init(&ifull[r], 1);
      tc::mbar_init(&iempty[r], (PAIR && !leader) ? 1 + G : 2 + G);  // producer, [MMA,] epilogues
    }
    for (int b = 0; b < 4; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], (PAIR ? 2 : 1) * G * TC_M);  // pair: both CTAs' epilogues
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&dfull[b], 1);
      tc::mbar_init(&dempty[b], (PAIR ? 2 : 1) * G * TC_M);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmA1);
    if (has_lo) tc::tma_prefetch(&tmA2);
    tc::tma_prefetch(PAIR ? &tmB1h : &tmB1);
    tc::tma_prefetch(PAIR ? &tmB2h : &tmB2);
  }
  if (warp == 1) {
    if (PAIR)
      tc::tmem_alloc_2sm<TMEM_COLS>(tmem_holder);
    else
      tc::tmem_alloc<TMEM_COLS>(tmem_holder);
  }
  tc::tc_fence_before();
  if (PAIR) tc::cluster_sync(); else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    // (L2 evict-first hints on the postings measured slower: a posting tile
    // is re-read by the next probe tile of its cell)
    // whole warp runs the loop (warp-uniform operands), one elected lane issues
    {
      int stage = 0;
      uint32_t phase = 0, it = 0;
      for (;; ++it) {  // items from the scheduler until its stop entry
        const uint32_t slot = it % ITEM_RING, iph = (it / ITEM_RING) & 1;
        tc::mbar_wait(&ifull[slot], iph);
        const ItemInfo I = s_item[slot];
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&iempty[slot]);
        if (I.c < 0) break;
        if (lane == 0) GIFT_TRACE(p, it, 1, clock64());
        const int brows = PAIR ? I.n / 2 : I.n;            // probe rows per plane half
        const uint32_t a_bytes = has_lo ? 2 * A_TILE : A_TILE;
        // this CTA's B bytes: both planes (single), one whole plane (pair, cb),
        // half of each plane (pair, lo)
        const uint32_t bytes =
            a_bytes + (PAIR && qz ? brows : PAIR && cb ? I.n : (qz ? 1 : 2) * brows) * TC_BK * 2;
        for (int kb = 0; kb < nkb; kb += kps) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * st_bytes;
          const int nk = min(kps, nkb - kb);  // k-blocks in this stage
          if (!tc::elect_one()) {
            // other lanes: nothing to issue
          } else if (GIFT_EXP(p, 8)) {
            if (!PAIR || leader) tc::mbar_arrive(&full[stage]);
          } else if (PAIR) {
            // both CTAs' bytes complete on the leader's full barrier
            const uint32_t lbar = tc::mapa(&full[stage], 0);
            if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * bytes);
            tc::tma_load_2d_2sm(st, &tmA1, lbar, kb * TC_BK, I.p0);
            if (has_lo) tc::tma_load_2d_2sm(st + A_TILE, &tmA2, lbar, kb * TC_BK, I.p0);
            const int r0 = I.pb0 + static_cast<int>(rank) * brows;
            if (qz) {  // fp16-exact queries: CTA r holds its half of b1's rows
              tc::tma_load_2d_2sm(st + b_off, brows == 64 ? &tmB1 : &tmB1h, lbar, kb * TC_BK, r0);
            } else if (cb) {  // CTA r: plane r, all n probe rows
              const CUtensorMap* pm = rank == 0 ? &tmB1 : &tmB2;
              for (int x = 0; x < I.n / 64; ++x)
                tc::tma_load_2d_2sm(st + b_off + x * B_BOX, pm, lbar, kb * TC_BK,
                                    I.pb0 + 64 * x);
            } else if (brows == 64) {
              tc::tma_load_2d_2sm(st + b_off, &tmB1, lbar, kb * TC_BK, r0);
              tc::tma_load_2d_2sm(st + b_off + B_PART, &tmB2, lbar, kb * TC_BK, r0);
            } else {
              tc::tma_load_2d_2sm(st + b_off, &tmB1h, lbar, kb * TC_BK, r0);
              tc::tma_load_2d_2sm(st + b_off + B_PART, &tmB2h, lbar, kb * TC_BK, r0);
            }
          } else if (small_st) {  // [A(kb) | b1(kb)] [A(kb+1) | b1(kb+1)]
            tc::mbar_arrive_expect_tx(&full[stage], nk * bytes);
            for (int j = 0; j < nk; ++j) {
              uint8_t* sj = st + j * SUB;
              tc::tma_load_2d(sj, &tmA1, &full[stage], (kb + j) * TC_BK, I.p0);
              for (int x = 0; x < I.n / 64; ++x)
                tc::tma_load_2d(sj + A_TILE + x * B_BOX, &tmB1, &full[stage], (kb + j) * TC_BK,
                                I.pb0 + 64 * x);
            }
          } else {
            tc::mbar_arrive_expect_tx(&full[stage], bytes);
            tc::tma_load_2d(st, &tmA1, &full[stage], kb * TC_BK, I.p0);
            if (has_lo) tc::tma_load_2d(st + A_TILE, &tmA2, &full[stage], kb * TC_BK, I.p0);
            // B1 rows then B2 rows back to back: one N = 2n MMA operand [b1 | b2]
            for (int x = 0; x < I.n / 64; ++x) {
              tc::tma_load_2d(st + b_off + x * B_BOX, &tmB1, &full[stage], kb * TC_BK,
                              I.pb0 + 64 * x);
              if (!qz)
                tc::tma_load_2d(st + b_off + I.n * TC_BK * 2 + x * B_BOX, &tmB2, &full[stage],
                                kb * TC_BK, I.pb0 + 64 * x);
            }
          }
          __syncwarp();
          if (++stage == n_st) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) GIFT_TRACE(p, it, 2, clock64());
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    // (pair: the leader issues cta_group::2 MMAs for both CTAs)
    // The whole warp runs the loop (waits, descriptor arithmetic: warp-uniform
    // values); one elected lane issues the MMAs and commits.
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t chunk_ctr = 0, item_ctr = 0;
      for (;;) {
        const uint32_t slot = item_ctr % ITEM_RING, sph = (item_ctr / ITEM_RING) & 1;
        tc::mbar_wait(&ifull[slot], sph);
        const ItemInfo I = s_item[slot];
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&iempty[slot]);
        if (I.c < 0) break;
        if (lane == 0) GIFT_TRACE(p, item_ctr, 3, clock64());
        const uint32_t idesc = tc::idesc_f16_f32(PAIR ? 2 * TC_M : TC_M, I.n);
        const uint32_t idesc2 = tc::idesc_f16_f32(PAIR ? 2 * TC_M : TC_M, 2 * I.n);  // [b1 | b2]
        const uint32_t ib = item_ctr & 1, iph = (item_ctr >> 1) & 1;
        uint32_t d2 = 0;
        if (!cb) {
          tc::mbar_wait(&dempty[ib], iph ^ 1);  // D2 buffer of this item free
          tc::tc_fence_after();
          d2 = tmem_base + 256 + ib * TC_NMAX;
        }
        for (int kb0 = 0; kb0 < nkb; kb0 += chunk_kb) {
          const uint32_t buf = chunk_ctr % nbuf, aph = (chunk_ctr / nbuf) & 1;
          tc::mbar_wait(&tempty[buf], aph ^ 1);
          tc::tc_fence_after();
          // pair: D1 per chunk buffer, D2 per item; single: [D1 | D2] per chunk
          // buffer; qz4: D1 per chunk buffer
          const uint32_t d1 = tmem_base + buf * buf_cols;
          const int kend = min(kb0 + chunk_kb, nkb);
          for (int kb = kb0; kb < kend; kb += kps) {
            tc::mbar_wait(&full[stage], phase);
            tc::tc_fence_after();
            uint8_t* st = smem + stage * st_bytes;
            if (small_st) {  // fp16-exact queries, single CTA: D1 = a1 . b1, kps k-blocks
              const int nk = min(kps, kend - kb);
              if (tc::elect_one()) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                  if (j >= nk) break;
                  const uint64_t a1 = tc::smem_desc_sw128(st + j * SUB);
                  const uint64_t b1 = tc::smem_desc_sw128(st + j * SUB + A_TILE);
#pragma unroll
                  for (int k = 0; k < TC_BK / 16; ++k) {
                    if (GIFT_EXP(p, 4)) break;
                    const uint32_t acc1 = (kb + j > kb0 || k > 0) ? 1u : 0u;
                    const uint64_t adv = static_cast<uint64_t>(k * 2);
                    tc::mma_f16(d1, a1 + adv, b1 + adv, idesc, acc1);
                  }
                }
                tc::mma_commit(&empty[stage]);
              }
              __syncwarp();
              if (++stage == n_st) {
                stage = 0;
                phase ^= 1;
              }
              continue;
            }
            const uint64_t a1 = tc::smem_desc_sw128(st);
            const uint64_t a2 = tc::smem_desc_sw128(st + A_TILE);
            const uint64_t b1 = tc::smem_desc_sw128(st + b_off);
            const uint64_t b2 = tc::smem_desc_sw128(st + b_off + B_PART);
            if (tc::elect_one()) {
#pragma unroll
              for (int k = 0; k < TC_BK / 16; ++k) {
                if (GIFT_EXP(p, 4)) break;
                const uint32_t acc1 = (kb > kb0 || k > 0) ? 1u : 0u;
                const uint32_t acc2 = (kb > 0 || k > 0) ? 1u : 0u;
                const uint64_t adv = static_cast<uint64_t>(k * 2);  // 32 B in 16-B units
                if (PAIR && qz) {  // D1 = a1 . b1, M = 256, b1 split over the pair
                  tc::mma_f16_2sm(d1, a1 + adv, b1 + adv, idesc, acc1);
                } else if (PAIR && cb) {  // [D1 | D2] = a1 . [b1 | b2], M = 256
                  tc::mma_f16_2sm(d1, a1 + adv, b1 + adv, idesc2, acc1);
                } else if (PAIR) {
                  tc::mma_f16_2sm(d1, a1 + adv, b1 + adv, idesc, acc1);
                  tc::mma_f16_2sm(d2, a1 + adv, b2 + adv, idesc, acc2);
                  tc::mma_f16_2sm(d2, a2 + adv, b1 + adv, idesc, 1u);
                } else if (qz) {  // b2 = 0: D1 = a1 . b1 [, D2 = a2 . b1]
                  tc::mma_f16(d1, a1 + adv, b1 + adv, idesc, acc1);
                  if (has_lo) tc::mma_f16(d1 + I.n, a2 + adv, b1 + adv, idesc, acc1);
                } else {
                  // a1 . [b1 | b2] -> [D1 | D2] (A read once), then D2 += a2 . b1
                  tc::mma_f16(d1, a1 + adv, b1 + adv, idesc2, acc1);
                  if (has_lo) tc::mma_f16(d1 + I.n, a2 + adv, b1 + adv, idesc, 1u);
                }
              }
              if (PAIR) tc::mma_commit_2sm(&empty[stage], 0x3); else tc::mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == n_st) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (tc::elect_one()) {
            if (PAIR) tc::mma_commit_2sm(&tfull[buf], 0x3); else tc::mma_commit(&tfull[buf]);
          }
          __syncwarp();
          ++chunk_ctr;
        }
        if (!cb && tc::elect_one()) tc::mma_commit_2sm(&dfull[ib], 0x3);
        __syncwarp();
        if (lane == 0) GIFT_TRACE(p, item_ctr, 4, clock64());
        ++item_ctr;
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------ scheduler
    // decodes the work items ahead of the other roles (the cell search and
    // tile lookups are dependent global loads that would otherwise stall the
    // MMA issuer between items)
    // Items are taken from a global counter (meta[M_WORK], zeroed by the
    // plan kernel) as CTAs become free, so the probe tiles of one posting
    // tile (consecutive items) run at the same time on neighbouring SMs and
    // the posting tile's re-reads hit L2 (a static stride lets the CTAs drift
    // apart); GIFT_FIF_SCHED_STATIC restores the stride.  Pair: the leader
    // fetches and pushes each index into the peer's s_next ring.
    if (lane == 0) {
      int hint = 0;
      unsigned long long* work =
          reinterpret_cast<unsigned long long*>(const_cast<int64_t*>(p.meta) + M_WORK);
      const uint32_t peer_next = PAIR ? tc::mapa(&s_next[0], 1) : 0u;
      const uint32_t peer_full = PAIR ? tc::mapa(&xfull[0], 1) : 0u;
      const uint32_t lead_empty = PAIR ? tc::mapa(&xempty[0], 0) : 0u;
      for (uint32_t it = 0;; ++it) {
        const uint32_t slot = it % ITEM_RING, iph = (it / ITEM_RING) & 1;
        int64_t item;
        if (!PAIR || leader) {
          item = p.dyn ? static_cast<int64_t>(atomicAdd(work, 1ull))
                       : first + static_cast<int64_t>(it) * stride;
          if (PAIR) {
            tc::mbar_wait(&xempty[slot], iph ^ 1);  // the peer took this slot's last index
            tc::st_cluster_u64(peer_next + slot * 8, item);
            tc::mbar_arrive_cluster(peer_full + slot * 8);
          }
        } else {
          tc::mbar_wait_cluster(&xfull[slot], iph);
          item = s_next[slot];
          tc::mbar_arrive_cluster(lead_empty + slot * 8);
        }
        ItemInfo I;
        if (item < n_items) {
          I = decode_item<PAIR>(p, item, hint, rank);
        } else {
          I.c = -1;  // stop entry for every role
        }
        tc::mbar_wait(&iempty[slot], iph ^ 1);
        s_item[slot] = I;
        tc::mbar_arrive(&ifull[slot]);
        GIFT_TRACE(p, it, 0, clock64());
        if (item < n_items) {
          GIFT_TRACE(p, it, 8, I.n);
          GIFT_TRACE(p, it, 9, I.c);
        }
        if (item >= n_items) break;
      }
    }
  } else {
    // ------------------------------------------------------ epilogue
    // G groups of 4 warps; group eg drains and reduces probe columns
    // [eg n / G, (eg + 1) n / G) of every item
    const int et = threadIdx.x - 96;      // 0 .. 128 G - 1
    const int eg = et >> 7;               // column group
    const int e = et & (TC_M - 1);        // thread within the group
    const int bar_tail = 1 + 2 * eg, bar_item = 2 + 2 * eg;
    constexpr int EC = Epi<G>::COLS, ES = Epi<G>::STRIDE;
    float* Dg = Ds + eg * Epi<G>::DS;
    int32_t* sp_s = s_sp + eg * (TC_M + 2);
    const int lb = 32 * (warp & 3);       // TMEM lane quarter of this warp
    const int row = lb + lane;            // posting row within the tile
    const bool gauss = p.mode == GIFT_SIM_GAUSSIAN;
    uint32_t chunk_ctr = 0, item_ctr = 0;
    // accumulator release: own barrier, or the pair leader's (remote arrive)
    const uint32_t rel_d0 = PAIR ? tc::mapa(&dempty[0], 0) : 0u;
    const uint32_t rel_d1 = PAIR ? tc::mapa(&dempty[1], 0) : 0u;
    for (;;) {
      const uint32_t slot = item_ctr % ITEM_RING, sph = (item_ctr / ITEM_RING) & 1;
      tc::mbar_wait(&ifull[slot], sph);
      const ItemInfo I = s_item[slot];
      named_bar(bar_item, TC_M);  // every thread of the group has its copy
      if (e == 0) tc::mbar_arrive(&iempty[slot]);
      if (I.c < 0) break;
      if (et == 0) GIFT_TRACE(p, item_ctr, 5, clock64());
      const int nseg = I.seg1 - I.seg0;
      const int hn = I.n / G;     // this group's columns: [c0, c0 + hn)
      const int c0 = eg * hn;
      const int ng = hn / 16;     // its 16-column groups
      // tail inputs, loaded now and staged to shared memory only at the tail
      // (their latency overlaps the drains): segment starts (nseg + 1 <= 129)
      // and the probe-sorted |q|^2
      const int sp_a = e <= nseg ? p.seg_pstart[I.seg0 + e] : 0;
      const int sp_b = e + TC_M <= nseg ? p.seg_pstart[I.seg0 + e + TC_M] : 0;
      const float qn_r = (e < hn && c0 + e < I.nb) ? p.qn2s[I.pb0 + c0 + e] : 0.f;
      // the row's |p|^2 and the cell's output coordinates, loaded now too
      // (posting-indexed |p|^2 misses L2: its latency would sit in the tail)
      const float pn = (gauss && I.p0 + row < I.p1) ? p.pnorm2[I.p0 + row] : 0.f;
      const int64_t seg_base = p.seg_off[I.c];
      const int64_t S_c = p.seg_off[I.c + 1] - seg_base;
      const int64_t obase = p.outbase[I.c];
      constexpr int NA = TC_NMAX / G;
      float acc[NA];
#pragma unroll
      for (int n = 0; n < NA; ++n) acc[n] = 0.f;
      const uint32_t lane_off = static_cast<uint32_t>(lb) << 16;
      for (int kb0 = 0; kb0 < nkb; kb0 += chunk_kb) {
        const uint32_t buf = chunk_ctr % nbuf, aph = (chunk_ctr / nbuf) & 1;
        tc::mbar_wait(&tfull[buf], aph);
        tc::tc_fence_after();
        if (!cb) {
          const uint32_t base = tmem_base + lane_off + buf * TC_NMAX + c0;
#pragma unroll
          for (int j = 0; j < NA / 16; j += 2) {
            if (j < ng && !GIFT_EXP(p, 2)) {
              float v1[16], v2[16];
              tc::tmem_ld_x16(base + j * 16, v1);
              tc::tmem_ld_x16(base + (j + 1) * 16, v2);  // ng is even
              tc::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                acc[j * 16 + i] += v1[i];
                acc[(j + 1) * 16 + i] += v2[i];
              }
            }
          }
        } else if (qz4) {  // D1 only: acc += D1
          const uint32_t base = tmem_base + lane_off + buf * TC_NMAX + c0;
#pragma unroll
          for (int j = 0; j < NA / 16; j += 2) {
            if (j < ng && !GIFT_EXP(p, 2)) {
              float v1[16], v2[16];
              tc::tmem_ld_x16(base + j * 16, v1);
              tc::tmem_ld_x16(base + (j + 1) * 16, v2);  // ng is even
              tc::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                acc[j * 16 + i] += v1[i];
                acc[(j + 1) * 16 + i] += v2[i];
              }
            }
          }
        } else {  // [D1 | D2] of this chunk: acc += D1 + 2^-11 D2
          const uint32_t base = tmem_base + lane_off + buf * 2 * TC_NMAX + c0;
#pragma unroll
          for (int j = 0; j < NA / 16; ++j) {
            if (j < ng && !GIFT_EXP(p, 2)) {
              float v1[16], v2[16];
              tc::tmem_ld_x16(base + j * 16, v1);
              tc::tmem_ld_x16(base + I.n + j * 16, v2);
              tc::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) acc[j * 16 + i] += fmaf(v2[i], SPLIT_INV, v1[i]);
            }
          }
        }
        tc::tc_fence_before();
        if (PAIR)
          tc::mbar_arrive_cluster_relaxed(tc::mapa(&tempty[buf], 0));  // the leader's barrier
        else
          tc::mbar_arrive_relaxed(&tempty[buf]);
        ++chunk_ctr;
      }
      if (cb) {
        ++item_ctr;
      } else {  // the item's correction terms, once: acc += 2^-11 D2
        const uint32_t ib = item_ctr & 1, iph = (item_ctr >> 1) & 1;
        tc::mbar_wait(&dfull[ib], iph);
        tc::tc_fence_after();
        const uint32_t base = tmem_base + lane_off + 256 + ib * TC_NMAX + c0;
#pragma unroll
        for (int j = 0; j < NA / 16; j += 2) {
          if (j < ng) {
            float v1[16], v2[16];
            tc::tmem_ld_x16(base + j * 16, v1);
            tc::tmem_ld_x16(base + (j + 1) * 16, v2);
            tc::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              acc[j * 16 + i] = fmaf(v1[i], SPLIT_INV, acc[j * 16 + i]);
              acc[(j + 1) * 16 + i] = fmaf(v2[i], SPLIT_INV, acc[(j + 1) * 16 + i]);
            }
          }
        }
        tc::tc_fence_before();
        if (PAIR)
          tc::mbar_arrive_cluster_relaxed(ib ? rel_d1 : rel_d0);
        else
          tc::mbar_arrive_relaxed(&dempty[ib]);
        ++item_ctr;
      }
      if (et == 0) GIFT_TRACE(p, item_ctr - 1, 6, clock64());
      if (p.tcomp_scale != 0.f) {  // add back the expected truncation loss
#pragma unroll
        for (int n = 0; n < NA; ++n) acc[n] = fmaf(acc[n], p.tcomp_scale, acc[n]);
      }
      if (!I.live || GIFT_EXP(p, 1)) {  // pair: duplicate tile, nothing to write
        named_bar(bar_tail, TC_M);
        continue;
      }
      if (e <= nseg) sp_s[e] = sp_a;
      if (e + TC_M <= nseg) sp_s[e + TC_M] = sp_b;
      if (e < hn) s_qn2[eg * TC_NMAX + c0 + e] = qn_r;
      // thread -> (column mc = e % EC, segments e / EC, + TC_M / EC, ...)
      const int mc = e & (EC - 1), sg0 = e / EC;
      // EC-column slices: stage -> per-segment max over rows -> store
#pragma unroll
      for (int sl0 = 0; sl0 < NA; sl0 += EC) {
        if (sl0 < hn && c0 + sl0 < I.nb) {
#pragma unroll
          for (int c = 0; c < EC; ++c) {
            float v = acc[sl0 + c];
            if (gauss) v = 2.0f * v - pn;  // max_p(2q.p - |p|^2) <-> min_p |q-p|^2
            Dg[row * ES + c] = v;
          }
          named_bar(bar_tail, TC_M);
          const int ncol = min(EC, I.nb - (c0 + sl0));
          const int m = c0 + sl0 + mc;
          for (int sl = sg0; mc < ncol && sl < nseg; sl += TC_M / EC) {
            const int sp0 = sp_s[sl], sp1 = sp_s[sl + 1];
            const int r0 = max(sp0, I.p0) - I.p0, r1 = min(sp1, I.p1) - I.p0;
            float mx = -INFINITY;
            for (int r = r0; r < r1; ++r) mx = fmaxf(mx, Dg[r * ES + mc]);
            float sim;
            if (gauss)
              sim = expf(-fmaxf(s_qn2[eg * TC_NMAX + m] - mx, 0.f) * p.inv_sigma2);
            else
              sim = fminf(fmaxf(mx, 0.f), 1.f);
            const int64_t o = obase + static_cast<int64_t>(I.mt * TC_NMAX + m) * S_c +
                              (I.seg0 + sl - seg_base);
            if (sp0 < I.p0 || sp1 > I.p1) {
              atomicMax(reinterpret_cast<int*>(p.out + o), __float_as_int(sim));
            } else {
              p.out[o] = sim;
            }
          }
          named_bar(bar_tail, TC_M);
        }
      }
      if (et == 0) GIFT_TRACE(p, item_ctr - 1, 7, clock64());
    }
  }
  tc::tc_fence_before();
  if (PAIR) tc::cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    if (PAIR)
      tc::tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
    else
      tc::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

__global__ void split_planes_kernel(const float* __restrict__ x, int64_t n, __half* __restrict__ h1,
                                    __half* __restrict__ h2) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (; i < n; i += stride) {
    __half a, b;
    split2(x[i], a, b);
    h1[i] = a;
    h2[i] = b;
  }
}

// Sorted probe rows -> query planes: G[s] = split(Q[probe_list[s] / ma]).
__global__ void probe_gather_split_kernel(const float* __restrict__ Q, int d, int ma,
                                          const int32_t* __restrict__ probe_list,
                                          const int32_t* __restrict__ probe_off, int K,
                                          const int64_t* __restrict__ meta,
                                          __half* __restrict__ g1, __half* __restrict__ g2,
                                          const float* __restrict__ qn2,
                                          float* __restrict__ qn2s) {
  if (meta[M_OVERFLOW]) return;
  const int s = blockIdx.x;
  if (s >= probe_off[K]) return;
  const int64_t view = probe_list[s] / ma;
  if (threadIdx.x == 0) qn2s[s] = qn2[view];  // |q|^2 in probe order (scan epilogue)
  const float* q = Q + view * d;
  __half* o1 = g1 + static_cast<int64_t>(s) * d;
  __half* o2 = g2 + static_cast<int64_t>(s) * d;
  bool lo = false;
  for (int k = threadIdx.x * 4; k < d; k += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(q + k);
    __half a0, a1, a2, a3, b0, b1, b2, b3;
    split2(v.x, a0, b0);
    split2(v.y, a1, b1);
    split2(v.z, a2, b2);
    split2(v.w, a3, b3);
    reinterpret_cast<__half2*>(o1 + k)[0] = __halves2half2(a0, a1);
    reinterpret_cast<__half2*>(o1 + k)[1] = __halves2half2(a2, a3);
    reinterpret_cast<__half2*>(o2 + k)[0] = __halves2half2(b0, b1);
    reinterpret_cast<__half2*>(o2 + k)[1] = __halves2half2(b2, b3);
    lo |= (__half_as_ushort(b0) | __half_as_ushort(b1) | __half_as_ushort(b2) |
           __half_as_ushort(b3)) & 0x7fff;
  }
  if (__syncthreads_or(lo) && threadIdx.x == 0)
    atomicOr(reinterpret_cast<unsigned long long*>(const_cast<int64_t*>(meta) + M_QLO), 1ull);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t d, uint32_t box_rows) {
  auto fn = encode_fn();
  GIFT_REQUIRE(fn != nullptr, GIFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {d, rows};
  cuuint64_t strides[1] = {d * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(TC_BK), box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  GIFT_REQUIRE(r == CUDA_SUCCESS, GIFT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return GIFT_OK;
}

size_t tc_probe_plane_bytes(int64_t nprobes, int d) {
  return align_up(static_cast<size_t>(nprobes) * d * 2, 1024);
}

bool tc_supported(const gift_fif_view* f) {
  return f->feat_hi != nullptr && f->d % 8 == 0 && f->d >= 8 && f->n_postings > 0;
}

// CTA pairs by default with the f32 lo plane (configs 2/3: half the L2 -> smem
// traffic per SM; config 3 scan 16.3 -> 15.1 ms, config 2 unchanged); fp16
// storage: the dense cells on the probe-major pair kernel (fif_scan_dense.cu),
// the others on single CTAs (the posting-major pair is ~7% slower there)
// persistent scan CTAs: one per SM minus the view's GIFT_FIF_RESERVE_SMS
// (left to the kernels of other batches in flight)
static int scan_ctas(const gift_fif_view* f) {
  const int reserve = (f->flags >> 8) & 255;
  return max(2, sm_count() - reserve);
}

bool tc_pair_enabled(const gift_fif_view* f) {
  const int m = (f->flags >> GIFT_FIF_PAIR_SHIFT) & 3;
  if (m == GIFT_FIF_PAIR_OFF) return false;
  if (m == GIFT_FIF_PAIR_ON) return sm_count() >= 2;
  return f->feat_lo != nullptr && sm_count() >= 2;
}

// fp16 storage, default pairing, segments within tiles: the dense cells run
// on the probe-major pair kernel, the rest on the single-CTA kernel
bool tc_dense_enabled(const gift_fif_view* f) {
  return f->feat_lo == nullptr && !(f->flags & GIFT_FIF_DENSE_OFF) &&
         (f->flags & GIFT_FIF_TILED_SEGMENTS) &&
         ((f->flags >> GIFT_FIF_PAIR_SHIFT) & 3) == GIFT_FIF_PAIR_AUTO && sm_count() >= 2;
}

template <int G, bool LO>
static cudaError_t launch_pair(int ctas, cudaStream_t st, const CUtensorMap& mA1,
                               const CUtensorMap& mA2, const CUtensorMap& mB1,
                               const CUtensorMap& mB2, const CUtensorMap& mB1h,
                               const CUtensorMap& mB2h, const TcArgs& a) {
  cudaError_t e = cudaFuncSetAttribute(fif_scan_tc_kernel<true, G, LO>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, Epi<G>::SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(max(2, ctas / 2 * 2)));
  cfg.blockDim = dim3(Epi<G>::THREADS);
  cfg.dynamicSmemBytes = Epi<G>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fif_scan_tc_kernel<true, G, LO>, mA1, mA2, mB1, mB2, mB1h, mB2h,
                            a);
}

int launch_scan_tc(const gift_fif_view* f, const float* Q, int64_t nprobes_max, TcArgs a,
                   __half* g1, __half* g2, cudaStream_t st, void* ev0, void* ev1) {
  const int d = f->d;
  const bool pair = tc_pair_enabled(f);
  probe_gather_split_kernel<<<static_cast<unsigned>(max64(nprobes_max, 1)), 128, 0, st>>>(
      Q, d, a.ma, a.probe_list, a.probe_off, f->K, a.meta, g1, g2, a.qn2, a.qn2s);
  GIFT_LAUNCH_CHECK();
  CUtensorMap mA1, mA2, mB1, mB2, mB1h, mB2h;
  int rc = make_map(&mA1, f->feat_hi, f->n_postings, d, TC_M);
  if (rc) return rc;
  rc = make_map(&mA2, f->feat_lo ? f->feat_lo : f->feat_hi, f->n_postings, d, TC_M);
  if (rc) return rc;
  rc = make_map(&mB1, g1, max64(nprobes_max, 1), d, 64);
  if (rc) return rc;
  rc = make_map(&mB2, g2, max64(nprobes_max, 1), d, 64);
  if (rc) return rc;
  rc = make_map(&mB1h, g1, max64(nprobes_max, 1), d, 32);
  if (rc) return rc;
  rc = make_map(&mB2h, g2, max64(nprobes_max, 1), d, 32);
  if (rc) return rc;
  a.has_lo = f->feat_lo != nullptr ? 1 : 0;
  if (ev0) GIFT_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(ev0), st));
  if (tc_dense_enabled(f)) {  // dense cells first (exits at once without dense items)
    CUtensorMap mQ;
    rc = make_map(&mQ, g1, max64(nprobes_max, 1), d, 128);
    if (rc) return rc;
    GIFT_CUDA_TRY(launch_scan_dense(scan_ctas(f), st, mQ, mA1, a, a.item_off2));
  }
  if (pair && a.has_lo) {
    GIFT_CUDA_TRY((launch_pair<1, true>(scan_ctas(f), st, mA1, mA2, mB1, mB2, mB1h, mB2h, a)));
  } else if (pair) {  // fp16 storage: tensor-bound, two epilogue groups
    GIFT_CUDA_TRY((launch_pair<2, false>(scan_ctas(f), st, mA1, mA2, mB1, mB2, mB1h, mB2h, a)));
  } else if (a.has_lo) {
    GIFT_CUDA_TRY((cudaFuncSetAttribute(fif_scan_tc_kernel<false, 2, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Epi<2>::SMEM)));
    fif_scan_tc_kernel<false, 2, true><<<scan_ctas(f), Epi<2>::THREADS, Epi<2>::SMEM, st>>>(
        mA1, mA2, mB1, mB2, mB1h, mB2h, a);
  } else {
    GIFT_CUDA_TRY((cudaFuncSetAttribute(fif_scan_tc_kernel<false, 2, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Epi<2>::SMEM)));
    fif_scan_tc_kernel<false, 2, false><<<scan_ctas(f), Epi<2>::THREADS, Epi<2>::SMEM, st>>>(
        mA1, mA2, mB1, mB2, mB1h, mB2h, a);
  }
  GIFT_LAUNCH_CHECK();
  if (ev1) GIFT_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(ev1), st));
  return GIFT_OK;
}

}  // namespace gift

using namespace gift;

extern "C" int gift_split_planes(const float* x, int64_t n, void* h1, void* h2, void* stream) {
  if (n <= 0) return GIFT_OK;
  split_planes_kernel<<<static_cast<unsigned>(min64(cdiv(n, 256), 8192)), 256, 0,
                        as_stream(stream)>>>(x, n, static_cast<__half*>(h1),
                                             static_cast<__half*>(h2));
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

#ifdef GIFT_SCAN_EXPERIMENT
namespace gift {
int g_scan_experiment = 0;
}
extern "C" void gift_scan_experiment(int bits) { gift::g_scan_experiment = bits; }
namespace gift {
unsigned long long* g_scan_trace = nullptr;
}
extern "C" void gift_scan_trace(void* buf) {
  gift::g_scan_trace = static_cast<unsigned long long*>(buf);
}
#endif
