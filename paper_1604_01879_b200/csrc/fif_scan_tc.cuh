// Shared declarations of the two F-IF scan implementations (fif_scan.cu,
// fif_scan_tc.cu).
#pragma once
#include <cuda.h>

#include "gift_common.cuh"

namespace gift {

// meta[M_QLO] != 0: some probe's query lo plane (b2) is non-zero.  Queries
// whose values are exactly fp16 (config 4's fp16-rounded views) leave it 0 and
// the single-CTA scan then skips the b2 operand (half the MMA work, bit-identical).
// M_ITEMS2 / M_WORK2: the dense-cell scan's item list (fif_scan_dense.cu).
enum Meta { M_ITEMS = 0, M_OUT_TOTAL = 1, M_OVERFLOW = 2, M_WORK = 3, M_QLO = 4, M_ITEMS2 = 5,
            M_WORK2 = 6 };

struct TcArgs {
  const int64_t* item_off;
  const int64_t* item_off2;  // dense-cell items (fif_scan_dense.cu)
  const int32_t* counts;
  const int32_t* probe_off;
  const int32_t* probe_list;
  const int64_t* outbase;
  float* out;
  const int64_t* meta;
  const int64_t* tile_off;
  const int32_t* tile_pstart;
  const int32_t* tile_pend;
  const int32_t* tile_seg0;
  const int32_t* tile_seg1;
  const int64_t* seg_off;
  const int32_t* seg_pstart;
  const float* pnorm2;
  const float* qn2;
  float* qn2s;  // [nprobes] |q|^2 in probe (cell-major) order, written by the gather
  int K, d, ma, mode;
  float inv_sigma2;
  int has_lo;
  int chunk_kb;
  int dyn;       // items from the meta[M_WORK] counter (1) or a static CTA stride (0)
  float tcomp_scale;  // acc *= 1 + tcomp_scale after the drains (0: no compensation)
#ifdef GIFT_SCAN_EXPERIMENT
  int exp;  // timing experiments only (tools/scan_experiment.py): 1 = no epilogue tail,
            // 2 = no TMEM drains, 4 = no MMAs, 8 = no loads; outputs invalid
  unsigned long long* trace;  // per-role clock64 stamps of the first CTAs' items (or null)
#endif
};

// Truncation compensation.  The tensor cores' fp32 accumulation truncates
// (measured: every scan score low, the bias linear in the MMA steps per
// drain: -3.4e-6 relative on gaussian scores at 16 steps, std ~0.2e-6;
// tools/drain_error.py).  A K = 16 step loses on average half an ulp of the
// running accumulator; a drained chunk v = m 2^e (m in [1, 2)) reached by n
// steps of roughly even increments has lost about 0.5 n ulp(v) (1 - 2/(3m)),
// i.e. a fraction 0.5 n 2^-23 (1/m)(1 - 2/(3m)) of v, whose mean over
// log-uniform mantissas is 0.5 n 2^-23 / (4 ln 2).  The chunks' shares of a
// dot scale with their lengths, so each item's dots are scaled once by
//   1 + TCOMP_PER_STEP * sum_c n_c^2 r(n_c) / sum_c n_c.
// r(n) is the measured excess of the loss over that model (the loss per
// step grows with the chain: 1.2x at 4 steps .. 1.8x at 64), calibrated
// against the f64 oracle on fp16 storage (c4s) and f32 planes (c2s) alike
// (tools/drain_error.py, profiles/r02/drain_interval_error_study.jsonl:
// uncompensated gaussian-score bias -0.72/-0.80, -1.55/-1.67, -3.44/-3.64,
// -8.05/-8.06, -17.7/-17.4 e-6 at 4, 8, 16, 32, 64 steps per chunk).
constexpr double TCOMP_PER_STEP = 0.5 * 0x1p-23 / (4.0 * 0.6931471805599453);
inline double tcomp_ratio(double n) {
  constexpr double R[5] = {1.22, 1.30, 1.43, 1.63, 1.77};  // n = 4, 8, 16, 32, 64
  const double x = log2(n < 4 ? 4.0 : n > 64 ? 64.0 : n) - 2.0;  // 0 .. 4
  const int i = x >= 4.0 ? 3 : static_cast<int>(x);
  return R[i] + (R[i + 1] - R[i]) * (x - i);
}

#ifdef GIFT_SCAN_EXPERIMENT
#define GIFT_EXP(p, bit) (((p).exp & (bit)) != 0)
// per-role clock64 stamps of the first CTAs' items (tools/scan_trace.py):
// trace[((cta * TR_ITEMS) + item) * TR_F + field]
constexpr int TR_CTAS = 8, TR_ITEMS = 512, TR_F = 16;
// (the dense-cell kernel stamps the second half: GIFT_TRACE_K(p, 1, ...))
#define GIFT_TRACE_K(p, k, it, f, v)                                                  \
  do {                                                                                \
    if ((p).trace != nullptr && blockIdx.x < TR_CTAS && (it) < TR_ITEMS)              \
      (p).trace[(((k) * TR_CTAS + blockIdx.x) * TR_ITEMS + (it)) * TR_F + (f)] = (v); \
  } while (0)
#define GIFT_TRACE(p, it, f, v) GIFT_TRACE_K(p, 0, it, f, v)
#else
#define GIFT_EXP(p, bit) false
#define GIFT_TRACE(p, it, f, v) do {} while (0)
#define GIFT_TRACE_K(p, k, it, f, v) do {} while (0)
#endif

bool tc_supported(const gift_fif_view* f);
// The scan on CTA pairs (cta_group::2, M = 256): a work item is two
// consecutive posting tiles of a cell x one probe tile.  GIFT_FIF_PAIR(m) in
// the view flags overrides the default (pairs with the f32 lo plane).
bool tc_pair_enabled(const gift_fif_view* f);
// quantize with need_order = false: when exactly ma candidates survive the
// margin test their order is not resolved (the F-IF scan takes a max over
// the ma cells, matching.py:153-159, so only the set matters)
int quantize_impl(const void* X, int32_t xdtype, int64_t n, int32_t d, const float* C,
                  const double* cnorm2, int32_t K, double cmax_norm, int32_t ma,
                  const uint8_t* nz, int32_t zero_key, int32_t* out_idx, void* ws,
                  size_t ws_bytes, void* stream, bool need_order, const float* xnorm2,
                  bool allow_tc);
size_t tc_probe_plane_bytes(int64_t nprobes, int d);
// Dense cells of an fp16-storage index (>= DENSE_MIN_PROBES probes in the
// batch, fp16-exact queries): probe-major CTA-pair scan (fif_scan_dense.cu).
constexpr int DENSE_MIN_PROBES = 192;
bool tc_dense_enabled(const gift_fif_view* f);
cudaError_t launch_scan_dense(int ctas, cudaStream_t st, const CUtensorMap& mQ,
                              const CUtensorMap& mP, const TcArgs& a, const int64_t* item_off2);
int launch_scan_tc(const gift_fif_view* f, const float* Q, int64_t nprobes_max, TcArgs a,
                   __half* g1, __half* g2, cudaStream_t st, void* ev0, void* ev1);

// tensor-core stage 1 of quantize (quant_tc.cu)
double tc_dot_eps(int d);
bool quant_tc_supported(int d, int xdtype);
size_t quant_tc_ws_bytes(int64_t rows, int d, int K);
int quant_approx_tc(const void* X, int xdtype, int64_t n, int d, const float* C, int K,
                    float* part, int ksplit_max, int* ksplit_out, void* ws, size_t ws_bytes,
                    cudaStream_t st);

}  // namespace gift
