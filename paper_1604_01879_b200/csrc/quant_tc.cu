// K1 stage 1 on the tensor cores: partial dots  part[z][v][c] = x_v . c_c over
// the z-th k-split, with the same fp16 two-plane operands as the tcgen05 scan
// (x = h1 + 2^-11 h2; per k-step one N = 256 MMA x1 . [c1 | c2] -> [D1 | D2]
// over the back-to-back centroid planes (x1 read once) and, with the query lo
// plane, D2 += x2 . c1; fp32 TMEM accumulators drained to registers every 4
// k-blocks).  The select stage (quantize.cu) widens its margin by the error
// coefficient `tc_dot_eps()` so the exact re-check still decides every
// assignment bit-exactly.
//
// Tiles: M = 128 vectors x N = 128 centroids; warp 0 TMA, warp 1 MMA, warps
// 2..9 epilogue in two column groups (same roles as fif_scan_tc.cu); producer
// and MMA loops run
// warp-wide and issue from one elected lane (descriptors stay uniform).
#include <cudaTypedefs.h>

#include "fif_scan_tc.cuh"
#include "tc_ptx.cuh"

namespace gift {

namespace {
constexpr int QM = 128, QN = 128, QBK = 64, QSTAGES = 3;
constexpr int QA_TILE = QM * QBK * 2;  // 16 KB
constexpr int QB_TILE = QN * QBK * 2;  // 16 KB
constexpr int QSTAGE = 2 * QA_TILE + 2 * QB_TILE;
constexpr int QEG = 2;                    // epilogue groups of 4 warps (QN / QEG columns each)
constexpr int QNG = QN / QEG;
constexpr int QTHREADS = 64 + 128 * QEG;
constexpr uint32_t QTMEM = 512;  // [D1 | D2] x 2 chunk buffers
constexpr int QSMEM = QSTAGES * QSTAGE + 256;
constexpr int QCHUNK_KB = 4;
constexpr float QSPLIT_INV = 1.0f / 2048.0f;
}  // namespace

struct QuantTcArgs {
  int64_t n;
  int K, d, ksplit, kchunk_kb, has_lo;
  float* part;  // [ksplit][n][K]
};

__global__ void __launch_bounds__(QTHREADS, 1)
    quant_approx_tc_kernel(const __grid_constant__ CUtensorMap tmX1,
                           const __grid_constant__ CUtensorMap tmX2,
                           const __grid_constant__ CUtensorMap tmC1,
                           const __grid_constant__ CUtensorMap tmC2, const QuantTcArgs p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + QSTAGES * QSTAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + QSTAGES;
  uint64_t* tfull = bars + 2 * QSTAGES;
  uint64_t* tempty = bars + 2 * QSTAGES + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * QSTAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t mt = (p.n + QM - 1) / QM;
  const int nt = (p.K + QN - 1) / QN;
  const int64_t n_items = mt * nt * p.ksplit;
  const int nkb_total = (p.d + QBK - 1) / QBK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < QSTAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], QEG * QM);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmX1);
    if (p.has_lo) tc::tma_prefetch(&tmX2);
    tc::tma_prefetch(&tmC1);
    tc::tma_prefetch(&tmC2);
  }
  if (warp == 1) tc::tmem_alloc<QTMEM>(tmem_holder);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // item -> (row tile, col tile, k split)
  auto decode = [&](int64_t item, int64_t& r0, int& c0, int& kb0, int& kb1) {
    const int z = static_cast<int>(item % p.ksplit);
    const int64_t rest = item / p.ksplit;
    c0 = static_cast<int>(rest % nt) * QN;
    r0 = (rest / nt) * QM;
    kb0 = z * p.kchunk_kb;
    kb1 = min(nkb_total, kb0 + p.kchunk_kb);
  };

  if (warp == 0) {
    {
      const uint32_t bytes = (p.has_lo ? 2 * QA_TILE : QA_TILE) + 2 * QB_TILE;
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        int64_t r0;
        int c0, kb0, kb1;
        decode(item, r0, c0, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * QSTAGE;
          if (tc::elect_one()) {
            tc::mbar_arrive_expect_tx(&full[stage], bytes);
            tc::tma_load_2d(st, &tmX1, &full[stage], kb * QBK, static_cast<int32_t>(r0));
            if (p.has_lo)
              tc::tma_load_2d(st + QA_TILE, &tmX2, &full[stage], kb * QBK,
                              static_cast<int32_t>(r0));
            tc::tma_load_2d(st + 2 * QA_TILE, &tmC1, &full[stage], kb * QBK, c0);
            tc::tma_load_2d(st + 2 * QA_TILE + QB_TILE, &tmC2, &full[stage], kb * QBK, c0);
          }
          __syncwarp();
          if (++stage == QSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {
      const uint32_t idesc = tc::idesc_f16_f32(QM, QN);
      const uint32_t idesc2 = tc::idesc_f16_f32(QM, 2 * QN);  // [c1 | c2]
      int stage = 0;
      uint32_t phase = 0, chunk_ctr = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        int64_t r0;
        int c0, kb0, kb1;
        decode(item, r0, c0, kb0, kb1);
        for (int ck = kb0; ck < kb1; ck += QCHUNK_KB) {
          const uint32_t buf = chunk_ctr & 1, aph = (chunk_ctr >> 1) & 1;
          tc::mbar_wait(&tempty[buf], aph ^ 1);
          tc::tc_fence_after();
          const uint32_t d1 = tmem_base + buf * 2 * QN, d2 = d1 + QN;
          const int kend = min(ck + QCHUNK_KB, kb1);
          for (int kb = ck; kb < kend; ++kb) {
            tc::mbar_wait(&full[stage], phase);
            tc::tc_fence_after();
            uint8_t* st = smem + stage * QSTAGE;
            const uint64_t a1 = tc::smem_desc_sw128(st);
            const uint64_t a2 = tc::smem_desc_sw128(st + QA_TILE);
            const uint64_t b1 = tc::smem_desc_sw128(st + 2 * QA_TILE);
            if (tc::elect_one()) {
#pragma unroll
              for (int k = 0; k < QBK / 16; ++k) {
                const uint32_t acc = (kb > ck || k > 0) ? 1u : 0u;
                const uint64_t adv = static_cast<uint64_t>(k * 2);
                tc::mma_f16(d1, a1 + adv, b1 + adv, idesc2, acc);  // [D1 | D2] = x1 . [c1 | c2]
                if (p.has_lo) tc::mma_f16(d2, a2 + adv, b1 + adv, idesc, 1u);
              }
              tc::mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == QSTAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (tc::elect_one()) tc::mma_commit(&tfull[buf]);
          __syncwarp();
          ++chunk_ctr;
        }
      }
    }
  } else {
    const int lb = 32 * (warp & 3);
    const int row = lb + lane;
    const int cg = (warp - 2) / 4 * QNG;  // this group's first column of the tile
    uint32_t chunk_ctr = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      int64_t r0;
      int c0, kb0, kb1;
      decode(item, r0, c0, kb0, kb1);
      const int z = static_cast<int>(item % p.ksplit);
      float acc[QNG];
#pragma unroll
      for (int c = 0; c < QNG; ++c) acc[c] = 0.f;
      for (int ck = kb0; ck < kb1; ck += QCHUNK_KB) {
        const uint32_t buf = chunk_ctr & 1, aph = (chunk_ctr >> 1) & 1;
        tc::mbar_wait(&tfull[buf], aph);
        tc::tc_fence_after();
        const uint32_t base =
            tmem_base + (static_cast<uint32_t>(lb) << 16) + buf * 2 * QN + cg;
#pragma unroll
        for (int j = 0; j < QNG / 16; ++j) {
          float v1[16], v2[16];
          tc::tmem_ld_x16(base + j * 16, v1);
          tc::tmem_ld_x16(base + QN + j * 16, v2);
          tc::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[j * 16 + i] += fmaf(v2[i], QSPLIT_INV, v1[i]);
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&tempty[buf]);
        ++chunk_ctr;
      }
      const int64_t v = r0 + row;
      if (v < p.n) {
        float* out = p.part + (static_cast<int64_t>(z) * p.n + v) * p.K + c0 + cg;
        const int nc = min(QNG, p.K - c0 - cg);
        if (nc == QNG && (p.K % 4) == 0) {
#pragma unroll
          for (int c = 0; c < QNG; c += 4)
            *reinterpret_cast<float4*>(out + c) =
                make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
        } else {
#pragma unroll
          for (int c = 0; c < QNG; ++c)
            if (c < nc) out[c] = acc[c];
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<QTMEM>(tmem_base);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 qencode_fn() {
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

static int qmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t d, uint32_t box_rows) {
  auto fn = qencode_fn();
  GIFT_REQUIRE(fn != nullptr, GIFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {d, rows};
  cuuint64_t strides[1] = {d * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(QBK), box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  GIFT_REQUIRE(r == CUDA_SUCCESS, GIFT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return GIFT_OK;
}

// Relative error coefficient of one tensor-core dot (vs |x| |c|): the split
// representation (<= 3 * 2^-22), <= 16 accumulator roundings per drained
// chunk (2^-23 each) and the fp32 sum of the drained chunks (2^-24 each, 16
// chunks at d = 4096), times a safety factor of 4.
double tc_dot_eps(int d) {
  const double nch = (d + QBK * QCHUNK_KB - 1) / (QBK * QCHUNK_KB) + 1.0;
  return 4.0 * (3.0 * 0x1p-22 + 4.0 * QCHUNK_KB * 0x1p-23 + nch * 0x1p-24);
}

bool quant_tc_supported(int d, int xdtype) {
  return d % 8 == 0 && d >= 8 && (xdtype == GIFT_F32 || xdtype == GIFT_F16);
}

size_t quant_tc_ws_bytes(int64_t rows, int d, int K) {
  return 2 * align_up(static_cast<size_t>(rows) * d * 2, 1024) +
         2 * align_up(static_cast<size_t>(K) * d * 2, 1024) + 4096;
}

int quant_approx_tc(const void* X, int xdtype, int64_t n, int d, const float* C, int K,
                    float* part, int ksplit_max, int* ksplit_out, void* ws, size_t ws_bytes,
                    cudaStream_t st) {
  Arena ar(ws, ws_bytes);
  const bool xhalf = xdtype == GIFT_F16;
  __half* x1 = xhalf ? static_cast<__half*>(const_cast<void*>(X)) : ar.take<__half>(n * d);
  __half* x2 = xhalf ? nullptr : ar.take<__half>(n * d);
  __half* c1 = ar.take<__half>(static_cast<int64_t>(K) * d);
  __half* c2 = ar.take<__half>(static_cast<int64_t>(K) * d);
  GIFT_REQUIRE(x1 && (xhalf || x2) && c1 && c2, GIFT_ERR_CAPACITY, "quantize workspace too small");
  int rc;
  if (!xhalf) {
    rc = gift_split_planes(static_cast<const float*>(X), n * d, x1, x2, st);
    if (rc) return rc;
  }
  rc = gift_split_planes(C, static_cast<int64_t>(K) * d, c1, c2, st);
  if (rc) return rc;
  // k-split so the grid covers the GPU; chunks are whole drain chunks
  const int nkb = (d + QBK - 1) / QBK;
  const int64_t tiles = cdiv(n, QM) * cdiv(K, QN);
  int ksplit = static_cast<int>(min64(cdiv(sm_count(), tiles), ksplit_max));
  ksplit = static_cast<int>(max64(1, min64(ksplit, cdiv(nkb, QCHUNK_KB))));
  int kchunk_kb = static_cast<int>(cdiv(cdiv(nkb, ksplit), QCHUNK_KB) * QCHUNK_KB);
  ksplit = static_cast<int>(cdiv(nkb, kchunk_kb));
  CUtensorMap mX1, mX2, mC1, mC2;
  if ((rc = qmap(&mX1, x1, n, d, QM))) return rc;
  if ((rc = qmap(&mX2, xhalf ? x1 : x2, n, d, QM))) return rc;
  if ((rc = qmap(&mC1, c1, K, d, QN))) return rc;
  if ((rc = qmap(&mC2, c2, K, d, QN))) return rc;
  QuantTcArgs a;
  a.n = n;
  a.K = K;
  a.d = d;
  a.ksplit = ksplit;
  a.kchunk_kb = kchunk_kb;
  a.has_lo = xhalf ? 0 : 1;
  a.part = part;
  GIFT_CUDA_TRY(cudaFuncSetAttribute(quant_approx_tc_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, QSMEM));
  const int64_t items = tiles * ksplit;
  quant_approx_tc_kernel<<<static_cast<unsigned>(min64(items, sm_count())), QTHREADS, QSMEM, st>>>(
      mX1, mX2, mC1, mC2, a);
  GIFT_LAUNCH_CHECK();
  *ksplit_out = ksplit;
  return GIFT_OK;
}

}  // namespace gift
