// Library plumbing: error state, scans, stable radix sort, offsets, view prep.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "gift_common.cuh"

namespace gift {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 148;
  }
  return cached;
}

// ---------------------------------------------------------------- scan
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename TIn>
__global__ void scan_tiles_kernel(const TIn* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                                  int64_t* __restrict__ tile_sums) {
  __shared__ int64_t sbuf[32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t local = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + i;
    v[i] = idx < n ? static_cast<int64_t>(in[idx]) : 0;
    local += v[i];
  }
  int64_t total;
  int64_t pre = block_exclusive_scan<int64_t>(local, &total, sbuf);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + i;
    if (idx < n) out[idx] = pre;
    pre += v[i];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

__global__ void scan_add_kernel(int64_t* __restrict__ out, int64_t n,
                                const int64_t* __restrict__ tile_prefix) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE;
  const int64_t add = tile_prefix[blockIdx.x];
  for (int i = threadIdx.x; i < SCAN_TILE; i += SCAN_THREADS) {
    int64_t idx = base + i;
    if (idx < n) out[idx] += add;
  }
}

__global__ void scan_total_kernel(const int64_t* ex_last, const int64_t* in64_last,
                                  const int32_t* in32_last, int64_t* dst) {
  *dst = *ex_last + (in64_last ? *in64_last : static_cast<int64_t>(*in32_last));
}

size_t scan_ws_bytes(int64_t n) {
  size_t total = 0;
  int64_t m = n;
  while (m > SCAN_TILE) {
    int64_t tiles = cdiv(m, SCAN_TILE);
    total += align_up(sizeof(int64_t) * (tiles + 1), 256);
    m = tiles;
  }
  return total + 256;
}

template <typename TIn>
static int scan_impl(const TIn* in, int64_t* out, int64_t n, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  if (n <= 0) return GIFT_OK;
  int64_t tiles = cdiv(n, SCAN_TILE);
  if (tiles == 1) {
    scan_tiles_kernel<TIn><<<1, SCAN_THREADS, 0, st>>>(in, out, n, nullptr);
    GIFT_LAUNCH_CHECK();
    return GIFT_OK;
  }
  Arena ar(ws, ws_bytes);
  int64_t* sums = ar.take<int64_t>(tiles + 1);
  GIFT_REQUIRE(sums != nullptr, GIFT_ERR_CAPACITY, "scan workspace too small");
  scan_tiles_kernel<TIn><<<static_cast<unsigned>(tiles), SCAN_THREADS, 0, st>>>(in, out, n, sums);
  GIFT_LAUNCH_CHECK();
  int rc = scan_impl<int64_t>(sums, sums, tiles, ar.base + ar.used, ar.remaining(), st);
  if (rc != GIFT_OK) return rc;
  scan_add_kernel<<<static_cast<unsigned>(tiles), SCAN_THREADS, 0, st>>>(out, n, sums);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

int scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, bool write_total, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  // The total needs the last input, which an in-place scan overwrites: stash it.
  Arena ar(ws, ws_bytes);
  int64_t* last = ar.take<int64_t>(1);
  GIFT_REQUIRE(last != nullptr, GIFT_ERR_CAPACITY, "scan workspace too small");
  if (write_total && n > 0)
    GIFT_CUDA_TRY(cudaMemcpyAsync(last, in + n - 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  int rc = scan_impl<int64_t>(in, out, n, ar.base + ar.used, ar.remaining(), st);
  if (rc != GIFT_OK) return rc;
  if (write_total) {
    if (n > 0) {
      scan_total_kernel<<<1, 1, 0, st>>>(out + n - 1, last, nullptr, out + n);
    } else {
      GIFT_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    }
    GIFT_LAUNCH_CHECK();
  }
  return GIFT_OK;
}

int scan_exclusive_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, bool write_total,
                              void* ws, size_t ws_bytes, cudaStream_t st) {
  int rc = scan_impl<int32_t>(in, out, n, ws, ws_bytes, st);
  if (rc != GIFT_OK) return rc;
  if (write_total) {
    if (n > 0)
      scan_total_kernel<<<1, 1, 0, st>>>(out + n - 1, nullptr, in + n - 1, out + n);
    else
      GIFT_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    GIFT_LAUNCH_CHECK();
  }
  return GIFT_OK;
}

// ---------------------------------------------------------------- radix sort
constexpr int RS_THREADS = 256;
constexpr int RS_ROUNDS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;  // items per block
constexpr int RS_WARPS = RS_THREADS / 32;

__global__ void radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                  int64_t nblk, int64_t* __restrict__ counts) {
  __shared__ int hist[256];
  hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
  for (int r = 0; r < RS_ROUNDS; ++r) {
    int64_t i = base + r * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&hist[(keys[i] >> shift) & 255u], 1);
  }
  __syncthreads();
  counts[static_cast<int64_t>(threadIdx.x) * nblk + blockIdx.x] = hist[threadIdx.x];
}

__global__ void radix_scatter_kernel(const uint32_t* __restrict__ keys_in,
                                     const uint32_t* __restrict__ vals_in,
                                     uint32_t* __restrict__ keys_out,
                                     uint32_t* __restrict__ vals_out, int64_t n, int shift,
                                     int64_t nblk, const int64_t* __restrict__ offsets) {
  __shared__ int64_t run_base[256];
  __shared__ int wcnt[RS_WARPS][257];
  __shared__ int wpre[RS_WARPS][257];
  __shared__ int tot[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  run_base[tid] = offsets[static_cast<int64_t>(tid) * nblk + blockIdx.x];
  for (int w = 0; w < RS_WARPS; ++w) wcnt[w][tid] = 0;
  if (tid == 0)
    for (int w = 0; w < RS_WARPS; ++w) wcnt[w][256] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int r = 0; r < RS_ROUNDS; ++r) {
    int64_t i = base + r * RS_THREADS + tid;
    bool valid = i < n;
    uint32_t key = valid ? keys_in[i] : 0u;
    uint32_t val = valid ? vals_in[i] : 0u;
    int digit = valid ? static_cast<int>((key >> shift) & 255u) : 256;
    unsigned peers = __match_any_sync(0xffffffffu, digit);
    int rank = __popc(peers & lt_mask);
    int leader = __ffs(peers) - 1;
    if (lane == leader) wcnt[warp][digit] = __popc(peers);
    __syncthreads();
    {
      int acc = 0;
      for (int w = 0; w < RS_WARPS; ++w) {
        int c = wcnt[w][tid];
        wpre[w][tid] = acc;
        acc += c;
      }
      tot[tid] = acc;
    }
    __syncthreads();
    if (valid) {
      int64_t pos = run_base[digit] + wpre[warp][digit] + rank;
      keys_out[pos] = key;
      vals_out[pos] = val;
    }
    __syncthreads();
    run_base[tid] += tot[tid];
    for (int w = 0; w < RS_WARPS; ++w) wcnt[w][tid] = 0;
    __syncthreads();
  }
}

}  // namespace gift

using namespace gift;

extern "C" size_t gift_radix_sort_ws_bytes(int64_t n) {
  int64_t nblk = cdiv(n > 0 ? n : 1, RS_TILE);
  return align_up(sizeof(int64_t) * (256 * nblk + 1), 256) + scan_ws_bytes(256 * nblk) + 1024;
}

extern "C" int gift_radix_sort_pairs(uint32_t* keys, uint32_t* vals, int64_t n, int32_t key_bits,
                                     uint32_t* keys_tmp, uint32_t* vals_tmp, void* ws,
                                     size_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n <= 1) return GIFT_OK;
  GIFT_REQUIRE(key_bits >= 0 && key_bits <= 32, GIFT_ERR_INVALID, "key_bits out of range");
  int64_t nblk = cdiv(n, RS_TILE);
  Arena ar(ws, ws_bytes);
  int64_t* counts = ar.take<int64_t>(256 * nblk + 1);
  GIFT_REQUIRE(counts != nullptr, GIFT_ERR_CAPACITY, "radix sort workspace too small");
  int passes = (key_bits + 7) / 8;
  uint32_t *kin = keys, *vin = vals, *kout = keys_tmp, *vout = vals_tmp;
  for (int p = 0; p < passes; ++p) {
    int shift = 8 * p;
    radix_hist_kernel<<<static_cast<unsigned>(nblk), RS_THREADS, 0, st>>>(kin, n, shift, nblk,
                                                                          counts);
    GIFT_LAUNCH_CHECK();
    int rc = scan_exclusive_i64(counts, counts, 256 * nblk, false, ar.base + ar.used,
                                ar.remaining(), st);
    if (rc != GIFT_OK) return rc;
    radix_scatter_kernel<<<static_cast<unsigned>(nblk), RS_THREADS, 0, st>>>(
        kin, vin, kout, vout, n, shift, nblk, counts);
    GIFT_LAUNCH_CHECK();
    uint32_t* t;
    t = kin; kin = kout; kout = t;
    t = vin; vin = vout; vout = t;
  }
  if (kin != keys) {
    GIFT_CUDA_TRY(cudaMemcpyAsync(keys, kin, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
    GIFT_CUDA_TRY(cudaMemcpyAsync(vals, vin, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  return GIFT_OK;
}

namespace gift {
__global__ void offsets_from_sorted_kernel(const uint32_t* __restrict__ keys, int64_t n,
                                           int64_t nb, int64_t* __restrict__ out) {
  int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b > nb) return;
  // lower_bound of b
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (static_cast<int64_t>(keys[mid]) < b)
      lo = mid + 1;
    else
      hi = mid;
  }
  out[b] = lo;
}

__global__ void view_prep_kernel(const void* __restrict__ X, int dtype, int64_t nviews, int d,
                                 uint8_t* __restrict__ nz, float* __restrict__ n2) {
  int64_t v = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (v >= nviews) return;
  double acc = 0.0;
  int any = 0;
  for (int k = lane; k < d; k += 32) {
    double x = load_as_f64(X, dtype, v * d + k);
    any |= (x != 0.0);
    acc += x * x;
  }
  any = __any_sync(0xffffffffu, any);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    if (nz) nz[v] = static_cast<uint8_t>(any);
    if (n2) n2[v] = static_cast<float>(acc);
  }
}

// GIFTFT1 ingest (features.py:67-71): row = (row_f64 / |row|) rounded to f32,
// rows with |row| == 0 copied unchanged.  |row| comes from the host (numpy's
// x.dot(x) of the reference, whose summation order belongs to its BLAS); the
// division and the rounding are IEEE here as there.
__global__ void normalize_rows_kernel(const float* x, const double* __restrict__ norms,
                                      int64_t rows, int d, float* out) {  // x may alias out
  const int64_t n = rows * d;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (; i < n; i += stride) {
    const double nr = norms[i / d];
    const float v = x[i];
    out[i] = nr == 0.0 ? v : __double2float_rn(__ddiv_rn(static_cast<double>(v), nr));
  }
}

__global__ void gather_rows_f32_kernel(const void* __restrict__ src, int dtype, int d,
                                       const int64_t* __restrict__ idx, int64_t n,
                                       float* __restrict__ out) {
  int64_t r = blockIdx.x;
  if (r >= n) return;
  int64_t s = idx[r];
  for (int k = threadIdx.x; k < d; k += blockDim.x)
    out[r * d + k] = load_as_f32(src, dtype, s * d + k);
}

__global__ void gather_rows_planes_kernel(const __half* __restrict__ hi,
                                          const __half* __restrict__ lo, int d,
                                          const int64_t* __restrict__ idx, int64_t n,
                                          float* __restrict__ out) {
  int64_t r = blockIdx.x;
  if (r >= n) return;
  int64_t s = idx[r];
  for (int k = threadIdx.x; k < d; k += blockDim.x)
    out[r * d + k] = __fadd_rn(__half2float(hi[s * d + k]),
                               __fmul_rn(__half2float(lo[s * d + k]), 1.0f / SPLIT_SCALE));
}
}  // namespace gift

extern "C" int gift_offsets_from_sorted(const uint32_t* keys, int64_t n, int64_t nbuckets,
                                        int64_t* out_off, void* stream) {
  cudaStream_t st = as_stream(stream);
  int64_t cnt = nbuckets + 1;
  offsets_from_sorted_kernel<<<static_cast<unsigned>(cdiv(cnt, 256)), 256, 0, st>>>(keys, n,
                                                                                   nbuckets, out_off);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_normalize_rows(const float* x, const double* norms, int64_t rows, int32_t d,
                                   float* out, void* stream) {
  GIFT_REQUIRE(rows >= 0 && d >= 1, GIFT_ERR_INVALID, "bad shape");
  if (rows == 0) return GIFT_OK;
  cudaStream_t st = as_stream(stream);
  normalize_rows_kernel<<<static_cast<unsigned>(min64(cdiv(rows * d, 256), 148 * 16)), 256, 0, st>>>(
      x, norms, rows, d, out);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_view_prep(const void* X, int32_t xdtype, int64_t nviews, int32_t d,
                              uint8_t* out_nz, float* out_norm2, void* stream) {
  if (nviews <= 0) return GIFT_OK;
  cudaStream_t st = as_stream(stream);
  view_prep_kernel<<<static_cast<unsigned>(cdiv(nviews, 8)), 256, 0, st>>>(X, xdtype, nviews, d,
                                                                          out_nz, out_norm2);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_gather_rows_f32(const void* src, int32_t dtype, int32_t d, const int64_t* idx,
                                    int64_t n, float* out, void* stream) {
  if (n <= 0) return GIFT_OK;
  cudaStream_t st = as_stream(stream);
  gather_rows_f32_kernel<<<static_cast<unsigned>(n), 128, 0, st>>>(src, dtype, d, idx, n, out);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_gather_rows_planes(const void* hi, const void* lo, int32_t d,
                                       const int64_t* idx, int64_t n, float* out, void* stream) {
  if (n <= 0) return GIFT_OK;
  cudaStream_t st = as_stream(stream);
  gather_rows_planes_kernel<<<static_cast<unsigned>(n), 128, 0, st>>>(
      static_cast<const __half*>(hi), static_cast<const __half*>(lo), d, idx, n, out);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_version(void) { return 1; }

extern "C" int gift_last_error(char* buf, size_t len) {
  if (buf && len) {
    strncpy(buf, gift::g_err, len - 1);
    buf[len - 1] = 0;
  }
  return GIFT_OK;
}
