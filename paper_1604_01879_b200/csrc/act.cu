// K5/K6 — sparse neighbour activations and the second inverted file.
// Replaces shapesearch.rerank (rerank.py:24-230).  Activations are kept in a
// fixed-capacity row format: idx[B, cap] (strictly ascending, -1 padded),
// val[B, cap] (f64 > 0), cnt[B], norm[B] (sequential ascending-coordinate f64
// sum, rerank.py:24-31, so a self-query's S-IF accumulator is bit-equal to
// the cached norm and scores exactly 1.0).
#include "gift_common.cuh"

namespace gift {

constexpr int MAX_NBR = 64;

__device__ __forceinline__ double seq_norm(const double* v, int n) {
  double t = 0.0;
  for (int i = 0; i < n; ++i) t = __dadd_rn(t, v[i]);
  return t;
}

// build_activation (rerank.py:64-75) + make_activation (:51-61): the first k1
// entries of a best-first top-k row that are present (idx >= 0, value > 0),
// re-ordered by ascending ordinal.  One warp per row.
__global__ void act_from_topk_kernel(const int32_t* __restrict__ tk_idx,
                                     const double* __restrict__ tk_val, int B, int kk, int k1,
                                     int cap, int32_t* __restrict__ a_idx,
                                     double* __restrict__ a_val, int32_t* __restrict__ a_cnt,
                                     double* __restrict__ a_norm) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const int lim = min(k1, kk);
  const int32_t* ti = tk_idx + b * kk;
  const double* tv = tk_val + b * kk;
  int n = 0;
  for (int i = 0; i < lim; ++i) n += (ti[i] >= 0 && tv[i] > 0.0) ? 1 : 0;
  int32_t* oi = a_idx + b * cap;
  double* ov = a_val + b * cap;
  for (int i = lane; i < cap; i += 32) {
    oi[i] = -1;
    ov[i] = 0.0;
  }
  __syncwarp();
  for (int i = lane; i < lim; i += 32) {
    const int32_t x = ti[i];
    if (x < 0 || !(tv[i] > 0.0)) continue;
    int rank = 0;
    for (int m = 0; m < lim; ++m) {
      const int32_t y = ti[m];
      if (y >= 0 && tv[m] > 0.0 && y < x) ++rank;
    }
    oi[rank] = x;
    ov[rank] = tv[i];
  }
  __syncwarp();
  if (lane == 0) {
    a_cnt[b] = n;
    a_norm[b] = seq_norm(ov, n);
  }
}

// mean_activation (rerank.py:90-100): dict accumulation in neighbour order,
// coordinates sorted, divided by len(neighbor_list).  One warp per row: the
// neighbours' sorted lists are staged in shared memory; an entry is the
// "first" of its coordinate if no earlier list holds it (binary search);
// first entries sum their coordinate over the lists in neighbour order (the
// reference's acc.get(idx, 0.0) + val sequence) and land at the rank of
// their coordinate among all first entries.
constexpr int AM_WARPS = 2;
constexpr int AM_MAX_E = 1024;

__device__ __forceinline__ bool list_has(const int32_t* idx, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (idx[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && idx[lo] == x;
}

__global__ void __launch_bounds__(AM_WARPS * 32)
    act_mean_kernel(const int32_t* __restrict__ raw_idx, const double* __restrict__ raw_val,
                    const int32_t* __restrict__ raw_cnt, int raw_cap,
                    const int32_t* __restrict__ nbr, int B, int k2, int cap,
                    int32_t* __restrict__ o_idx, double* __restrict__ o_val,
                    int32_t* __restrict__ o_cnt, double* __restrict__ o_norm) {
  __shared__ int32_t s_idx[AM_WARPS][AM_MAX_E];
  __shared__ double s_val[AM_WARPS][AM_MAX_E];
  __shared__ int16_t s_lst[AM_WARPS][AM_MAX_E];
  __shared__ int32_t s_first[AM_WARPS][AM_MAX_E];
  __shared__ int32_t s_off[AM_WARPS][MAX_NBR + 2];  // list ends [0, nl], nl at MAX_NBR + 1
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = static_cast<int64_t>(blockIdx.x) * AM_WARPS + warp;
  if (b >= B) return;
  int32_t* I = s_idx[warp];
  double* Vv = s_val[warp];
  int16_t* L = s_lst[warp];
  int32_t* F = s_first[warp];
  int32_t* off = s_off[warp];
  if (lane == 0) {
    int nl = 0, e = 0;
    off[0] = 0;
    for (int t = 0; t < k2; ++t) {
      const int q = nbr[b * k2 + t];
      if (q < 0) continue;
      e += raw_cnt[q];
      off[++nl] = e;
    }
    off[MAX_NBR + 1] = nl;
  }
  __syncwarp();
  const int nl = off[MAX_NBR + 1];
  const int E = off[nl];
  // stage the lists (list order = neighbour order)
  for (int t = 0, tt = 0; t < k2; ++t) {
    const int q = nbr[b * k2 + t];
    if (q < 0) continue;
    const int n0 = off[tt], n = off[tt + 1] - off[tt];
    for (int i = lane; i < n; i += 32) {
      I[n0 + i] = raw_idx[static_cast<int64_t>(q) * raw_cap + i];
      Vv[n0 + i] = raw_val[static_cast<int64_t>(q) * raw_cap + i];
      L[n0 + i] = static_cast<int16_t>(tt);
    }
    ++tt;
  }
  __syncwarp();
  for (int e = lane; e < E; e += 32) {
    const int x = I[e];
    bool first = true;
    for (int t = 0; t < L[e] && first; ++t)
      if (list_has(I + off[t], off[t + 1] - off[t], x)) first = false;
    F[e] = first ? 1 : 0;
  }
  __syncwarp();
  int32_t* oi = o_idx + b * cap;
  double* ov = o_val + b * cap;
  const double count = static_cast<double>(nl);
  int n_out = 0;
  for (int e = lane; e < E; e += 32) {
    if (!F[e]) continue;
    const int x = I[e];
    int rank = 0;
    for (int e2 = 0; e2 < E; ++e2) rank += (F[e2] && I[e2] < x) ? 1 : 0;
    double acc = 0.0;
    bool started = false;
    for (int t = L[e]; t < nl; ++t) {
      const int32_t* li = I + off[t];
      const int n = off[t + 1] - off[t];
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (li[mid] < x) lo = mid + 1; else hi = mid;
      }
      if (lo < n && li[lo] == x) {
        const double v = Vv[off[t] + lo];
        acc = started ? __dadd_rn(acc, v) : __dadd_rn(0.0, v);
        started = true;
      }
    }
    if (rank < cap) {
      oi[rank] = x;
      ov[rank] = __ddiv_rn(acc, count);
    }
  }
  for (int e = lane; e < E; e += 32) n_out += F[e];
  for (int o = 16; o > 0; o >>= 1) n_out += __shfl_xor_sync(0xffffffffu, n_out, o);
  __syncwarp();
  // raw values are > 0, so every mean is > 0 (make_activation keeps all)
  for (int i = n_out + lane; i < cap; i += 32) {
    oi[i] = -1;
    ov[i] = 0.0;
  }
  __syncwarp();
  if (lane == 0) {
    o_cnt[b] = min(n_out, cap);
    o_norm[b] = seq_norm(ov, min(n_out, cap));
  }
}

__device__ __forceinline__ double np_power_scalar(double v, double e) {
  // numpy: np.power(v, a) (libm pow) and ndarray ** e (fast paths for
  // e in {0.5, 1, 2}); the fast paths are exact/correctly rounded.
  if (e == 1.0) return v;
  if (e == 2.0) return __dmul_rn(v, v);
  if (e == 0.5) return __dsqrt_rn(v);
  return pow(v, e);
}

// aggregate (rerank.py:128-147): union support, equal values pass through.
__global__ void act_aggregate_kernel(const int32_t* __restrict__ ai, const double* __restrict__ av,
                                     const int32_t* __restrict__ ac, int acap,
                                     const int32_t* __restrict__ bi, const double* __restrict__ bv,
                                     const int32_t* __restrict__ bc, int bcap, int B, double alpha,
                                     int cap, int32_t* __restrict__ oi, double* __restrict__ ov,
                                     int32_t* __restrict__ oc, double* __restrict__ on) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int32_t* x = ai + b * acap;
  const double* xv = av + b * acap;
  const int32_t* y = bi + b * bcap;
  const double* yv = bv + b * bcap;
  const int nx = ac[b], ny = bc[b];
  int32_t* o = oi + b * cap;
  double* w = ov + b * cap;
  const double inv = 1.0 / alpha;
  int i = 0, j = 0, n = 0;
  while (i < nx || j < ny) {
    int idx;
    double v1 = 0.0, v2 = 0.0;
    if (j >= ny || (i < nx && x[i] < y[j])) {
      idx = x[i];
      v1 = xv[i++];
    } else if (i >= nx || y[j] < x[i]) {
      idx = y[j];
      v2 = yv[j++];
    } else {
      idx = x[i];
      v1 = xv[i++];
      v2 = yv[j++];
    }
    double r;
    if (v1 == v2) {
      r = v1;
    } else {
      const double s = __dadd_rn(np_power_scalar(v1, alpha), np_power_scalar(v2, alpha));
      r = np_power_scalar(__ddiv_rn(s, 2.0), inv);
    }
    if (r > 0.0 && n < cap) {
      o[n] = idx;
      w[n] = r;
      ++n;
    }
  }
  for (int k = n; k < cap; ++k) {
    o[k] = -1;
    w[k] = 0.0;
  }
  oc[b] = n;
  on[b] = seq_norm(w, n);
}

__global__ void act_compact_kernel(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                   const int32_t* __restrict__ cnt, int cap, int64_t nrows,
                                   const int64_t* __restrict__ row_off, uint32_t* __restrict__ key,
                                   uint32_t* __restrict__ pos, int32_t* __restrict__ owner,
                                   double* __restrict__ oval) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int64_t base = row_off[r];
  for (int e = 0; e < cnt[r]; ++e) {
    key[base + e] = static_cast<uint32_t>(idx[r * cap + e]);
    pos[base + e] = static_cast<uint32_t>(base + e);
    owner[base + e] = static_cast<int32_t>(r);
    oval[base + e] = val[r * cap + e];
  }
}

__global__ void sif_permute_kernel(const uint32_t* __restrict__ pos, const int32_t* __restrict__ owner,
                                   const double* __restrict__ val, int64_t nnz,
                                   int32_t* __restrict__ e_ord, double* __restrict__ e_val) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  const uint32_t p = pos[q];
  e_ord[q] = owner[p];
  e_val[q] = val[p];
}

// query_sif (rerank.py:211-230) for a batch: one CTA per query; the dense
// output row doubles as the accumulator.  Entries are visited in ascending
// coordinate order with a barrier between entries, so every acc[j] is the
// same left-to-right f64 sum as the reference's acc[ords] += min(...).
__global__ void __launch_bounds__(256)
    sif_query_kernel(const int64_t* __restrict__ e_off, const int32_t* __restrict__ e_ord,
                     const double* __restrict__ e_val, const double* __restrict__ norms,
                     int64_t n_global, int64_t n_local, const int32_t* __restrict__ q_idx,
                     const double* __restrict__ q_val, const int32_t* __restrict__ q_cnt,
                     const double* __restrict__ q_norm, int cap, double* __restrict__ out) {
  const int b = blockIdx.x;
  double* row = out + static_cast<int64_t>(b) * n_local;
  for (int64_t j = threadIdx.x; j < n_local; j += blockDim.x) row[j] = 0.0;
  __syncthreads();
  const int cnt = q_cnt[b];
  for (int e = 0; e < cnt; ++e) {
    const int64_t i = q_idx[static_cast<int64_t>(b) * cap + e];
    if (i < 0 || i >= n_global) continue;
    const double v = q_val[static_cast<int64_t>(b) * cap + e];
    const int64_t p0 = e_off[i], p1 = e_off[i + 1];
    for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
      const int32_t j = e_ord[p];
      row[j] = __dadd_rn(row[j], fmin(v, e_val[p]));
    }
    __syncthreads();
  }
  const double qn = q_norm[b];
  for (int64_t j = threadIdx.x; j < n_local; j += blockDim.x) {
    const double acc = row[j];
    if (acc > 0.0) row[j] = __ddiv_rn(acc, __dsub_rn(__dadd_rn(qn, norms[j]), acc));
  }
}

// query_sif + the final ranking (rerank.py:211-230, index.py:290-294) without
// the dense [B, n] row: a CTA serves queries b = blockIdx.x, + gridDim.x, ...
// with its own zero-initialised f64 accumulator row in global memory.  Entries
// are visited in ascending coordinate order with a barrier between entries
// (every acc[j] is the reference's left-to-right f64 sum); the first touch of
// j appends it to the query's candidate row.  Before the touched accumulators
// are finalised and cleared back to zero, one warp adds the zero-score fill
// the reference's lexsort would rank next: self (tiebreak 0) if untouched,
// then the first k untouched shapes by id rank.  The rows (score, tiebreak,
// global ordinal) go to the top-k merge pass, which ranks them exactly like
// the dense path (touched scores are > 0, so the fill only matters when fewer
// than k shapes are touched).
__global__ void __launch_bounds__(256)
    sif_query_sparse_kernel(const int64_t* __restrict__ e_off, const int32_t* __restrict__ e_ord,
                            const double* __restrict__ e_val, const double* __restrict__ norms,
                            int64_t n_global, int64_t n_local, const int32_t* __restrict__ q_idx,
                            const double* __restrict__ q_val, const int32_t* __restrict__ q_cnt,
                            const double* __restrict__ q_norm, int B, int cap,
                            double* __restrict__ acc_rows, int64_t acc_stride,
                            const int32_t* __restrict__ order,
                            const int32_t* __restrict__ idrank, const int32_t* __restrict__ self_local,
                            int64_t ord_base, int k_fill, int64_t m, double* __restrict__ cs,
                            uint32_t* __restrict__ ct, int32_t* __restrict__ ci,
                            int32_t* __restrict__ row_cnt) {
  __shared__ int s_cnt;
  double* acc = acc_rows + static_cast<int64_t>(blockIdx.x) * acc_stride;
  const int tid = threadIdx.x;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    const int64_t row = static_cast<int64_t>(b) * m;
    const int cnt = q_cnt[b];
    for (int e = 0; e < cnt; ++e) {
      const int64_t i = q_idx[static_cast<int64_t>(b) * cap + e];
      if (i < 0 || i >= n_global) continue;
      const double v = q_val[static_cast<int64_t>(b) * cap + e];
      const int64_t p0 = e_off[i], p1 = e_off[i + 1];
      for (int64_t p = p0 + tid; p < p1; p += blockDim.x) {
        const int32_t j = e_ord[p];
        const double old = acc[j];
        if (old == 0.0) ci[row + atomicAdd(&s_cnt, 1)] = j;  // contributions are > 0
        acc[j] = __dadd_rn(old, fmin(v, e_val[p]));
      }
      __syncthreads();
    }
    const int T = s_cnt;
    const int64_t sl = self_local ? static_cast<int64_t>(self_local[b]) : -1;
    if (tid < 32) {  // zero-score fill, one warp
      const int lane = tid;
      int pos = T;
      if (sl >= 0 && sl < n_local && acc[sl] == 0.0) {
        if (lane == 0) {
          cs[row + pos] = 0.0;
          ct[row + pos] = 0u;
          ci[row + pos] = static_cast<int32_t>(ord_base + sl);
        }
        ++pos;
      }
      int nf = 0;
      for (int64_t r0 = 0; nf < k_fill && r0 < n_local; r0 += 32) {
        const int64_t r = r0 + lane;
        int32_t j = -1;
        bool hit = false;
        if (r < n_local) {
          j = order[r];
          hit = j != sl && acc[j] == 0.0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        const int before = __popc(bal & ((1u << lane) - 1u));
        if (hit && nf + before < k_fill) {
          const int64_t at = row + pos + nf + before;
          cs[at] = 0.0;
          ct[at] = 1u + static_cast<uint32_t>(idrank ? static_cast<int64_t>(idrank[j]) : ord_base + j);
          ci[at] = static_cast<int32_t>(ord_base + j);
        }
        nf = min(k_fill, nf + __popc(bal));
      }
      if (lane == 0) row_cnt[b] = pos + nf;
    }
    __syncthreads();
    const double qn = q_norm[b];
    for (int t = tid; t < T; t += blockDim.x) {
      const int32_t j = ci[row + t];
      const double a = acc[j];
      acc[j] = 0.0;
      cs[row + t] = __ddiv_rn(a, __dsub_rn(__dadd_rn(qn, norms[j]), a));
      ct[row + t] = j == sl ? 0u
                            : 1u + static_cast<uint32_t>(idrank ? static_cast<int64_t>(idrank[j])
                                                                : ord_base + j);
      ci[row + t] = static_cast<int32_t>(ord_base + j);
    }
    __syncthreads();
  }
}

// ---- sort-based sparse S-IF query ----------------------------------------
// The same result as sif_query_sparse_kernel without per-query accumulator
// rows: every (query b, shape j, contribution) of the query's S-IF postings is
// emitted in entry order, the pairs are radix-sorted by (b, j) -- stable, so a
// shape's contributions keep ascending coordinate order -- and each run is
// summed sequentially from 0.0 (the reference's acc[j] += ... order,
// rerank.py:219-230).
__global__ void sif_tcount_kernel(const int32_t* __restrict__ q_idx,
                                  const int32_t* __restrict__ q_cnt, int cap,
                                  const int64_t* __restrict__ e_off, int64_t n_global, int B,
                                  int32_t* __restrict__ tcnt) {
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (b >= B) return;
  int64_t t = 0;
  for (int e = lane; e < q_cnt[b]; e += 32) {
    const int64_t i = q_idx[static_cast<int64_t>(b) * cap + e];
    if (i >= 0 && i < n_global) t += e_off[i + 1] - e_off[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) tcnt[b] = static_cast<int32_t>(t);
}

__global__ void __launch_bounds__(256)
    sif_emit_kernel(const int32_t* __restrict__ q_idx, const double* __restrict__ q_val,
                    const int32_t* __restrict__ q_cnt, int cap, const int64_t* __restrict__ e_off,
                    const int32_t* __restrict__ e_ord, const double* __restrict__ e_val,
                    int64_t n_global, int jbits, const int64_t* __restrict__ off,
                    uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                    double* __restrict__ contrib) {
  const int b = blockIdx.x;
  int64_t pos0 = off[b];
  for (int e = 0; e < q_cnt[b]; ++e) {
    const int64_t i = q_idx[static_cast<int64_t>(b) * cap + e];
    if (i < 0 || i >= n_global) continue;
    const double v = q_val[static_cast<int64_t>(b) * cap + e];
    const int64_t p0 = e_off[i], p1 = e_off[i + 1];
    for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
      const int64_t at = pos0 + (p - p0);
      keys[at] = (static_cast<uint32_t>(b) << jbits) | static_cast<uint32_t>(e_ord[p]);
      vals[at] = static_cast<uint32_t>(at);
      contrib[at] = fmin(v, e_val[p]);
    }
    pos0 += p1 - p0;
  }
}

// run-start flags, and the contributions gathered into sorted order (one
// independent load per thread instead of the run sums' dependent gathers)
__global__ void sif_runflag_kernel(const uint32_t* __restrict__ keys,
                                   const uint32_t* __restrict__ vals,
                                   const double* __restrict__ contrib, int64_t T,
                                   int32_t* __restrict__ flag, double* __restrict__ sorted) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= T) return;
  flag[t] = (t == 0 || keys[t - 1] != keys[t]) ? 1 : 0;
  sorted[t] = contrib[vals[t]];
}

// One thread per run start; rpos = exclusive scan of the run-start flags, so
// a query's runs fill its candidate row densely.
__global__ void sif_runsum_kernel(const uint32_t* __restrict__ keys,
                                  const uint32_t* __restrict__ vals,
                                  const double* __restrict__ contrib, int64_t T, int jbits,
                                  const int64_t* __restrict__ off, const int64_t* __restrict__ rpos,
                                  const double* __restrict__ norms,
                                  const double* __restrict__ q_norm,
                                  const int32_t* __restrict__ idrank,
                                  const int32_t* __restrict__ self_local, int64_t ord_base,
                                  int64_t m, double* __restrict__ cs, uint32_t* __restrict__ ct,
                                  int32_t* __restrict__ ci) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint32_t key = keys[t];
  if (t > 0 && keys[t - 1] == key) return;  // inside a run
  const int b = static_cast<int>(key >> jbits);
  const int32_t j = static_cast<int32_t>(key & ((1u << jbits) - 1u));
  const int64_t at = static_cast<int64_t>(b) * m + (rpos[t] - rpos[off[b]]);
  double a = 0.0;
  for (int64_t u = t; u < T && keys[u] == key; ++u) a = __dadd_rn(a, contrib[u]);
  const int64_t sl = self_local ? static_cast<int64_t>(self_local[b]) : -1;
  cs[at] = __ddiv_rn(a, __dsub_rn(__dadd_rn(q_norm[b], norms[j]), a));
  ct[at] = j == sl ? 0u
                   : 1u + static_cast<uint32_t>(idrank ? static_cast<int64_t>(idrank[j])
                                                        : ord_base + j);
  ci[at] = static_cast<int32_t>(ord_base + j);
}

// zero-score fill of sif_query_sparse_kernel (self first, then id-rank order)
// with "touched" = j present in the query's sorted run keys
__global__ void sif_fill_kernel(const uint32_t* __restrict__ keys, const int64_t* __restrict__ off,
                                const int64_t* __restrict__ rpos, int jbits, const int32_t* __restrict__ order,
                                const int32_t* __restrict__ idrank,
                                const int32_t* __restrict__ self_local, int64_t ord_base,
                                int64_t n_local, int k_fill, int B, int64_t m,
                                double* __restrict__ cs, uint32_t* __restrict__ ct,
                                int32_t* __restrict__ ci, int32_t* __restrict__ row_cnt) {
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (b >= B) return;
  const int64_t k0 = off[b], k1 = off[b + 1];
  const uint32_t hb = static_cast<uint32_t>(b) << jbits;
  auto touched = [&](int64_t j) {
    const uint32_t want = hb | static_cast<uint32_t>(j);
    int64_t lo = k0, hi = k1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < want) lo = mid + 1; else hi = mid;
    }
    return lo < k1 && keys[lo] == want;
  };
  const int64_t row = static_cast<int64_t>(b) * m;
  int64_t pos = rpos[k1] - rpos[k0];  // the query's touched shapes
  const int64_t sl = self_local ? static_cast<int64_t>(self_local[b]) : -1;
  if (sl >= 0 && sl < n_local && !touched(sl)) {
    if (lane == 0) {
      cs[row + pos] = 0.0;
      ct[row + pos] = 0u;
      ci[row + pos] = static_cast<int32_t>(ord_base + sl);
    }
    ++pos;
  }
  int nf = 0;
  for (int64_t r0 = 0; nf < k_fill && r0 < n_local; r0 += 32) {
    const int64_t r = r0 + lane;
    int32_t j = -1;
    bool hit = false;
    if (r < n_local) {
      j = order[r];
      hit = j != sl && !touched(j);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    const int before = __popc(bal & ((1u << lane) - 1u));
    if (hit && nf + before < k_fill) {
      const int64_t at = row + pos + nf + before;
      cs[at] = 0.0;
      ct[at] = 1u + static_cast<uint32_t>(idrank ? static_cast<int64_t>(idrank[j]) : ord_base + j);
      ci[at] = static_cast<int32_t>(ord_base + j);
    }
    nf = min(k_fill, nf + __popc(bal));
  }
  if (lane == 0) row_cnt[b] = static_cast<int32_t>(pos + nf);
}

// ---- bucketed S-IF query (no sort, no host synchronisation) ----------------
// The same result again, from a stable split of each query's pairs into
// buckets of 2^rb consecutive local shapes: one CTA per query counts its
// pairs per (warp, bucket) and scatters them warp-ordered, so every bucket
// holds its (shape, contribution) pairs in the query's entry order.  One warp
// then reduces a bucket in a dense f64 shared-memory accumulator; lanes of a
// 32-pair chunk that hit the same shape (two entries) take turns in lane
// order, so every sum is the reference's left-to-right acc[j] += ... order
// (rerank.py:219-230), bit-equal to the other two paths.
constexpr int SB_WARPS = 16;
constexpr int SB_MAX_R = 2048;  // buckets per query (split kernel counters)
constexpr int SB_MAX_E = 1024;  // query support entries staged in shared memory
// Bucket width and the reduce's occupancy (config 5, 1M shapes, 3 lanes;
// profiles/r02/c5_bucket_sweep_s4.txt): 2^11-shape buckets with one 13-warp
// CTA per SM 484k q/s; 2^10 with 2 / 3 / 4 CTAs per SM 516k / 517k / 524k;
// 2^9 (the split's per-bucket counters grow) 447-454k.
#ifndef GIFT_SB_MIN_RB
#define GIFT_SB_MIN_RB 10
#endif
#ifndef GIFT_SB_RED_KB
#define GIFT_SB_RED_KB 69
#endif
#ifndef GIFT_SB_RED_CTAS
#define GIFT_SB_RED_CTAS 3
#endif
constexpr int SB_MIN_RB = GIFT_SB_MIN_RB;  // 2^10 shapes (8 KB of f64) per reducing warp
constexpr int SB_RED_KB = GIFT_SB_RED_KB;      // shared accumulators per reducing CTA
constexpr int SB_RED_CTAS = GIFT_SB_RED_CTAS;  // reducing CTAs per SM
constexpr int SB_MAX_RB = 13;
#ifndef GIFT_SB_U
#define GIFT_SB_U 4
#endif
constexpr int SB_U = GIFT_SB_U;  // chunks of 32 pairs in flight per lane

// exclusive scan of a[0, n) in place (all threads of the CTA); returns the total
__device__ int32_t block_scan_excl(int32_t* a, int n, int32_t* wsum) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int i0 = min(n, tid * per), i1 = min(n, i0 + per);
  int32_t own = 0;
  for (int i = i0; i < i1; ++i) own += a[i];
  int32_t x = own;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int32_t before = 0, total = 0;
  for (int w = 0; w < nw; ++w) {
    if (w < warp) before += wsum[w];
    total += wsum[w];
  }
  int32_t run = before + x - own;
  for (int i = i0; i < i1; ++i) {
    const int32_t t = a[i];
    a[i] = run;
    run += t;
  }
  __syncthreads();
  return total;
}

__host__ __device__ constexpr size_t sb_align16(size_t x) { return (x + 15) / 16 * 16; }

size_t sif_split_smem(int cap, int R) {
  return static_cast<size_t>(cap) * 16 + sb_align16(sizeof(int32_t) * (cap + 1)) * 2 +
         sizeof(int32_t) * static_cast<size_t>(SB_WARPS + 1) * R;
}

// The entry holding chunk c: the last e >= e0 with cpre[e] <= c (warp-uniform;
// chunks of empty entries are skipped because their cpre equals the next one's).
__device__ __forceinline__ int chunk_entry(const int32_t* cpre, int ne, int e0, int32_t c,
                                           int lane) {
  for (;;) {
    const int e = e0 + lane;
    const unsigned m = __ballot_sync(0xffffffffu, e < ne && cpre[e] <= c);
    if (m != 0xffffffffu || e0 + 32 >= ne) return e0 + 31 - __clz(m);
    e0 += 32;
  }
}

// Persistent, one query per CTA at a time (queries b = blockIdx.x, + gridDim.x,
// ...: the output regions being filled stay few enough for L2 to merge their
// scattered writes).  The query's postings, entry by entry, form chunks of 32
// (entry-aligned); warp w owns a contiguous range of chunks.  Pass 1 counts
// pairs per (warp, bucket); the bucket starts plus the earlier warps' counts
// give every warp its own cursor per bucket; pass 2 scatters through them.  A
// chunk holds postings of one entry -- distinct shapes -- so the slot order
// inside a chunk is immaterial (an atomic ticket), while chunks, i.e.
// entries, stay in order (one warp's tickets in program order, a __syncwarp
// between chunks; warps in order of their ranges): every bucket lists each
// shape's contributions in entry order.
__global__ void __launch_bounds__(SB_WARPS * 32)
    sif_split_kernel(const int32_t* __restrict__ q_idx, const double* __restrict__ q_val,
                     const int32_t* __restrict__ q_cnt, int cap, int B,
                     const int64_t* __restrict__ e_off, const int32_t* __restrict__ e_ord,
                     const double* __restrict__ e_val, int64_t n_global, int rb, int R,
                     const int64_t* __restrict__ off, int32_t* __restrict__ bstart,
                     uint16_t* __restrict__ pj, double* __restrict__ pc) {
  extern __shared__ __align__(16) char sb_smem[];
  char* sp = sb_smem;
  int64_t* s_p0 = reinterpret_cast<int64_t*>(sp);
  sp += static_cast<size_t>(cap) * 8;
  double* s_v = reinterpret_cast<double*>(sp);
  sp += static_cast<size_t>(cap) * 8;
  int32_t* s_len = reinterpret_cast<int32_t*>(sp);
  sp += sb_align16(sizeof(int32_t) * (cap + 1));
  int32_t* s_cpre = reinterpret_cast<int32_t*>(sp);
  sp += sb_align16(sizeof(int32_t) * (cap + 1));
  int32_t* s_cnt = reinterpret_cast<int32_t*>(sp);  // [SB_WARPS][R]
  int32_t* s_tot = s_cnt + SB_WARPS * R;            // [R]
  __shared__ int32_t s_wsum[SB_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t mask = (1u << rb) - 1u;
  int32_t* my = s_cnt + warp * R;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const int ne = min(q_cnt[b], cap);
    for (int e = tid; e < ne; e += blockDim.x) {
      const int64_t i = q_idx[static_cast<int64_t>(b) * cap + e];
      const bool ok = i >= 0 && i < n_global;
      const int64_t a = ok ? e_off[i] : 0;
      const int32_t len = ok ? static_cast<int32_t>(e_off[i + 1] - a) : 0;
      s_p0[e] = a;
      s_v[e] = q_val[static_cast<int64_t>(b) * cap + e];
      s_len[e] = len;
      s_cpre[e] = (len + 31) >> 5;
    }
    for (int x = tid; x < SB_WARPS * R; x += blockDim.x) s_cnt[x] = 0;
    __syncthreads();
    const int32_t NC = block_scan_excl(s_cpre, ne, s_wsum);
    if (tid == 0) s_cpre[ne] = NC;
    __syncthreads();
    const int32_t per = (NC + SB_WARPS - 1) / SB_WARPS;
    const int32_t cw0 = min(NC, warp * per), cw1 = min(NC, cw0 + per);
    int e_first = 0;
    {  // last e with cpre[e] <= cw0 (same in every lane)
      int lo = 0, hi = max(ne - 1, 0);
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_cpre[mid] <= cw0) lo = mid; else hi = mid - 1;
      }
      e_first = lo;
    }
    // SB_U chunks' loads in flight (j = -1: no pair)
    auto load = [&](int32_t c0, int& e, int32_t (&jj)[SB_U], double (&cc)[SB_U],
                    double (&vq)[SB_U], bool vals) {
#pragma unroll
      for (int u = 0; u < SB_U; ++u) {
        const int32_t c = c0 + u;
        jj[u] = -1;
        if (c < cw1) {
          e = chunk_entry(s_cpre, ne, e, c, lane);
          const int32_t o = (c - s_cpre[e]) * 32 + lane;
          if (o < s_len[e]) {
            const int64_t p = s_p0[e] + o;
            jj[u] = e_ord[p];
            if (vals) {
              cc[u] = e_val[p];
              vq[u] = s_v[e];
            }
          }
        }
      }
    };
    {  // pass 1: per-(warp, bucket) counts
      int e = e_first;
      for (int32_t c0 = cw0; c0 < cw1; c0 += SB_U) {
        int32_t jj[SB_U];
        double cc[SB_U], vq[SB_U];
        load(c0, e, jj, cc, vq, false);
#pragma unroll
        for (int u = 0; u < SB_U; ++u)
          if (jj[u] >= 0) atomicAdd(&my[static_cast<uint32_t>(jj[u]) >> rb], 1);
      }
    }
    __syncthreads();
    int32_t* bs = bstart + static_cast<int64_t>(b) * (R + 1);
    for (int r = tid; r < R; r += blockDim.x) {  // per-warp offsets within a bucket
      int32_t run = 0;
      for (int w = 0; w < SB_WARPS; ++w) {
        const int32_t c = s_cnt[w * R + r];
        s_cnt[w * R + r] = run;
        run += c;
      }
      s_tot[r] = run;
    }
    __syncthreads();
    const int32_t tb = block_scan_excl(s_tot, R, s_wsum);  // bucket starts in the query's region
    for (int r = tid; r < R; r += blockDim.x) {
      const int32_t st = s_tot[r];
      bs[r] = st;
      for (int w = 0; w < SB_WARPS; ++w) s_cnt[w * R + r] += st;
    }
    if (tid == 0) bs[R] = tb;
    __syncthreads();
    {  // pass 2: the scatter
      const int64_t base = off[b];
      int e = e_first;
      for (int32_t c0 = cw0; c0 < cw1; c0 += SB_U) {
        int32_t jj[SB_U];
        double cc[SB_U], vq[SB_U];
        load(c0, e, jj, cc, vq, true);
#pragma unroll
        for (int u = 0; u < SB_U; ++u) {
          if (jj[u] >= 0) {
            const uint32_t j = static_cast<uint32_t>(jj[u]);
            const int32_t pos = atomicAdd(&my[j >> rb], 1);
            pj[base + pos] = static_cast<uint16_t>(j & mask);
            pc[base + pos] = fmin(vq[u], cc[u]);
          }
          __syncwarp();
        }
      }
    }
    __syncthreads();
  }
}

// Persistent: warp w reduces the contiguous bucket range [w per, (w + 1) per)
// (bucket g = query g / R, shape range g % R) in its shared f64 row
// acc[2^rb], zero between buckets.  The touched shapes' sums are compacted in
// place to the front of the bucket's pair region (pc = sum, pj = shape;
// count ntb[g]) -- the ranking kernel scores and selects them.  Bounds of 32
// buckets come in one load per lane; the next bucket's first chunk is loaded
// before the current one is reduced.
__global__ void sif_bucket_reduce_kernel(uint16_t* __restrict__ pj, double* __restrict__ pc,
                                         const int64_t* __restrict__ off,
                                         const int32_t* __restrict__ bstart, int B, int R, int rb,
                                         int32_t* __restrict__ ntb) {
  extern __shared__ double s_acc[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int W = 1 << rb;
  for (int x = tid; x < nw * W; x += blockDim.x) s_acc[x] = 0.0;
  __syncthreads();
  double* acc = s_acc + warp * W;
  const int64_t nb = static_cast<int64_t>(B) * R;
  const int64_t totw = static_cast<int64_t>(gridDim.x) * nw;
  const int64_t per = (nb + totw - 1) / totw;
  const int64_t g0 = (static_cast<int64_t>(blockIdx.x) * nw + warp) * per;
  const int64_t g1 = min64(nb, g0 + per);
  for (int64_t gb = g0; gb < g1; gb += 32) {
    int64_t sL = 0, eL = 0;
    if (gb + lane < g1) {
      const int64_t g = gb + lane;
      const int64_t b = g / R, r = g % R;
      const int64_t q0 = off[b];
      const int32_t* bs = bstart + b * (R + 1);
      sL = q0 + bs[r];
      eL = q0 + bs[r + 1];
    }
    const int nbk = static_cast<int>(min64(32, g1 - gb));
    int64_t s = __shfl_sync(0xffffffffu, sL, 0), e = __shfl_sync(0xffffffffu, eL, 0);
    uint32_t jn = s + lane < e ? pj[s + lane] : 0x10000u + lane;
    double cn = s + lane < e ? pc[s + lane] : 0.0;
    for (int i = 0; i < nbk; ++i) {
      // next bucket's bounds and first chunk
      const int64_t s2 = __shfl_sync(0xffffffffu, sL, (i + 1) & 31);
      const int64_t e2 = __shfl_sync(0xffffffffu, eL, (i + 1) & 31);
      const bool more = i + 1 < nbk;
      const uint32_t jn2 = more && s2 + lane < e2 ? pj[s2 + lane] : 0x10000u + lane;
      const double cn2 = more && s2 + lane < e2 ? pc[s2 + lane] : 0.0;
      int nt = 0;
      for (int64_t c0 = s; c0 < e; c0 += 32) {  // pass 1: accumulate in lane turns
        const uint32_t jl = jn;
        const double c = cn;
        const bool valid = c0 + lane < e;
        const int64_t tn = c0 + 32 + lane;
        jn = tn < e ? pj[tn] : 0x10000u + lane;
        cn = tn < e ? pc[tn] : 0.0;
        const unsigned peers = __match_any_sync(0xffffffffu, jl);
        const int rank = __popc(peers & lt);
        const int mr = __reduce_max_sync(0xffffffffu, rank);
        for (int rr = 0; rr <= mr; ++rr) {
          if (valid && rank == rr) acc[jl] = __dadd_rn(acc[jl], c);
          __syncwarp();
        }
      }
      for (int64_t c0 = s; c0 < e; c0 += 32) {  // pass 2: each shape once, compacted
        const int64_t t = c0 + lane;
        const bool valid = t < e;
        const uint32_t jl = valid ? pj[t] : 0x10000u + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, jl);
        const bool lead = valid && __ffs(peers) - 1 == lane;
        const double a = lead ? acc[jl] : 0.0;
        const bool fin = lead && a != 0.0;  // contributions are > 0
        if (fin) acc[jl] = 0.0;
        const unsigned fb = __ballot_sync(0xffffffffu, fin);
        if (fin) {  // slot <= t: pairs at or before this chunk, already read
          const int64_t at = s + nt + __popc(fb & lt);
          pc[at] = a;
          pj[at] = static_cast<uint16_t>(jl);
        }
        nt += __popc(fb);
        __syncwarp();
      }
      if (lane == 0) ntb[gb + i] = nt;
      s = s2;
      e = e2;
      jn = jn2;
      cn = cn2;
    }
  }
}

// Ranking of the bucketed query (index.py:290-294), one CTA per query: the
// touched shapes' (score, tiebreak, ordinal) -- the accumulator-row kernel's
// finalisation -- go to the query's candidate row at off[b] + b (k + 1),
// with the zero-score fill appended when fewer than k are touched.  Rows
// that fit the sort buffer are bitonic-sorted whole; longer rows are
// filtered by the k-th best of a strided sample (a lower bound of the row's
// k-th best key), survivors collected into the buffer in rounds that cannot
// overflow it and sorted with the running best.  Keys are unique per row, so
// the first k are the dense ranking's.
constexpr int RK_THREADS = 256;
constexpr int RK_BUF = 2048;  // sort buffer: [0, RK_BEST) best so far, then survivors
constexpr int RK_BEST = 256;  // >= k

__device__ void bitonic_sort_desc_n(double* s, uint32_t* t, int32_t* j, int N) {
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        const int lo = 2 * stride * (i / stride) + (i % stride);
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        if (key_better(s[hi], t[hi], s[lo], t[lo]) == desc) {
          const double ts = s[lo]; s[lo] = s[hi]; s[hi] = ts;
          const uint32_t tt = t[lo]; t[lo] = t[hi]; t[hi] = tt;
          const int32_t tj = j[lo]; j[lo] = j[hi]; j[hi] = tj;
        }
      }
      __syncthreads();
    }
  }
}

size_t sif_rank_smem(int R) { return static_cast<size_t>(RK_BUF) * 16 + sizeof(int32_t) * 2 * (R + 1); }

__global__ void __launch_bounds__(RK_THREADS)
    sif_bucket_rank_kernel(const uint16_t* __restrict__ pj, const double* __restrict__ pc,
                           const int64_t* __restrict__ off, const int32_t* __restrict__ bstart,
                           const int32_t* __restrict__ ntb, int R, int rb,
                           const double* __restrict__ norms, const double* __restrict__ q_norm,
                           const int32_t* __restrict__ order, const int32_t* __restrict__ idrank,
                           const int32_t* __restrict__ self_local, int64_t ord_base,
                           int64_t n_local, int k, double* __restrict__ cs,
                           uint32_t* __restrict__ ct, int32_t* __restrict__ ci,
                           int32_t* __restrict__ out_idx, double* __restrict__ out_val) {
  extern __shared__ __align__(16) char rk_smem[];
  double* xs = reinterpret_cast<double*>(rk_smem);
  uint32_t* xt = reinterpret_cast<uint32_t*>(rk_smem + RK_BUF * 8);
  int32_t* xj = reinterpret_cast<int32_t*>(rk_smem + RK_BUF * 12);
  int32_t* s_ps = reinterpret_cast<int32_t*>(rk_smem + RK_BUF * 16);  // pair starts
  int32_t* s_cs = s_ps + R + 1;                                         // candidate starts
  __shared__ int32_t s_wsum[RK_THREADS / 32];
  __shared__ int s_cnt, s_nfill;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int64_t q0 = off[b];
  const int64_t row = q0 + static_cast<int64_t>(b) * (k + 1);
  for (int r = tid; r <= R; r += RK_THREADS) {
    s_ps[r] = bstart[static_cast<int64_t>(b) * (R + 1) + r];
    s_cs[r] = r < R ? ntb[static_cast<int64_t>(b) * R + r] : 0;
  }
  if (tid == 0) s_nfill = 0;
  __syncthreads();
  const int32_t n = block_scan_excl(s_cs, R, s_wsum);
  if (tid == 0) s_cs[R] = n;
  __syncthreads();
  const double qn = q_norm[b];
  const int64_t sl = self_local ? static_cast<int64_t>(self_local[b]) : -1;
  const int32_t stride = n > RK_BUF ? (n + RK_BUF - 1) / RK_BUF : 1;
  // pass 1: score every touched shape (4 candidates' loads in flight per thread)
  for (int32_t t0 = 0; t0 < n; t0 += 4 * RK_THREADS) {
    double a[4], nr[4];
    int32_t jg[4], rk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t t = t0 + u * RK_THREADS + tid;
      jg[u] = -1;
      if (t < n) {
        int lo = 0, hi = R - 1;  // bucket: last r with s_cs[r] <= t
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_cs[mid] <= t) lo = mid; else hi = mid - 1;
        }
        const int64_t pos = q0 + s_ps[lo] + (t - s_cs[lo]);
        a[u] = pc[pos];
        jg[u] = (lo << rb) + pj[pos];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (jg[u] >= 0) {
        nr[u] = norms[jg[u]];
        rk[u] = idrank ? idrank[jg[u]] : 0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t t = t0 + u * RK_THREADS + tid;
      if (jg[u] < 0) continue;
      const int64_t j = jg[u];
      const double sc = __ddiv_rn(a[u], __dsub_rn(__dadd_rn(qn, nr[u]), a[u]));
      const uint32_t tb =
          j == sl ? 0u : 1u + static_cast<uint32_t>(idrank ? static_cast<int64_t>(rk[u]) : ord_base + j);
      const int32_t jj = static_cast<int32_t>(ord_base + j);
      cs[row + t] = sc;
      ct[row + t] = tb;
      ci[row + t] = jj;
      if (t % stride == 0) {
        const int32_t x = t / stride;
        xs[x] = sc;
        xt[x] = tb;
        xj[x] = jj;
      }
    }
  }
  __syncthreads();
  if (n < k && tid < 32) {  // zero-score fill (the whole row is in the buffer)
    const int lane = tid;
    auto touched = [&](int64_t j) {
      const int32_t want = static_cast<int32_t>(ord_base + j);
      for (int u = 0; u < n; ++u)
        if (xj[u] == want) return true;
      return false;
    };
    int pos = n;
    if (sl >= 0 && sl < n_local && !touched(sl)) {
      if (lane == 0) {
        cs[row + pos] = 0.0;
        ct[row + pos] = 0u;
        ci[row + pos] = static_cast<int32_t>(ord_base + sl);
      }
      ++pos;
    }
    int nf = 0;
    for (int64_t r0 = 0; nf < k && r0 < n_local; r0 += 32) {
      const int64_t r = r0 + lane;
      int32_t j = -1;
      bool hit = false;
      if (r < n_local) {
        j = order[r];
        hit = j != sl && !touched(j);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      const int before = __popc(bal & ((1u << lane) - 1u));
      if (hit && nf + before < k) {
        const int64_t at = row + pos + nf + before;
        cs[at] = 0.0;
        ct[at] = 1u + static_cast<uint32_t>(idrank ? static_cast<int64_t>(idrank[j]) : ord_base + j);
        ci[at] = static_cast<int32_t>(ord_base + j);
      }
      nf = min(k, nf + __popc(bal));
    }
    __syncwarp();
    // the appended entries into the buffer too
    for (int u = n + lane; u < pos + nf; u += 32) {
      xs[u] = cs[row + u];
      xt[u] = ct[row + u];
      xj[u] = ci[row + u];
    }
    if (lane == 0) s_nfill = pos + nf - n;
  }
  __syncthreads();
  const int ntot = n + s_nfill;
  auto pad_sort = [&](int from, int N) {
    for (int i = from + tid; i < N; i += RK_THREADS) {
      xs[i] = -INFINITY;
      xt[i] = 0xffffffffu;
      xj[i] = -1;
    }
    __syncthreads();
    bitonic_sort_desc_n(xs, xt, xj, N);
  };
  // the best-so-far plus survivors, sorted over the next power of two only
  // (the sorts are most of this kernel's instructions)
  auto pow2_at_least = [](int x) {
    int N = 2;
    while (N < x) N <<= 1;
    return N;
  };
  if (ntot <= RK_BUF) {
    int N = 2;
    while (N < ntot || N < k) N <<= 1;
    pad_sort(ntot, N);
  } else {
    pad_sort((n + stride - 1) / stride, RK_BUF);  // the sample
    double th_s = xs[k - 1];
    uint32_t th_t = xt[k - 1];
    __syncthreads();
    for (int i = tid; i < RK_BEST; i += RK_THREADS) {  // best: empty
      xs[i] = -INFINITY;
      xt[i] = 0xffffffffu;
      xj[i] = -1;
    }
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    int32_t t0 = 0;
    while (t0 < n) {
      const int cnt = s_cnt;
      const int free = RK_BUF - RK_BEST - cnt;
      if (free < 4 * RK_THREADS) {  // make room: keep the best RK_BEST
        __syncthreads();
        pad_sort(RK_BEST + cnt, pow2_at_least(RK_BEST + cnt));
        if (key_better(xs[k - 1], xt[k - 1], th_s, th_t)) {
          th_s = xs[k - 1];
          th_t = xt[k - 1];
        }
        __syncthreads();
        if (tid == 0) s_cnt = 0;
        __syncthreads();
        continue;
      }
      const int32_t span = min(free, n - t0);
      for (int32_t i0 = 0; i0 < span; i0 += 4 * RK_THREADS) {
        double sc[4];
        uint32_t tb[4];
        int32_t jj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int32_t i = i0 + u * RK_THREADS + tid;
          jj[u] = -1;
          if (i < span) {
            sc[u] = cs[row + t0 + i];
            tb[u] = ct[row + t0 + i];
            jj[u] = ci[row + t0 + i];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (jj[u] >= 0 && !key_better(th_s, th_t, sc[u], tb[u])) {
            const int p = RK_BEST + atomicAdd(&s_cnt, 1);
            xs[p] = sc[u];
            xt[p] = tb[u];
            xj[p] = jj[u];
          }
        }
      }
      t0 += span;
      __syncthreads();
    }
    pad_sort(RK_BEST + s_cnt, pow2_at_least(RK_BEST + s_cnt));
  }
  for (int i = tid; i < k; i += RK_THREADS) {
    const bool ok = xj[i] >= 0;
    out_idx[static_cast<int64_t>(b) * k + i] = ok ? xj[i] : -1;
    out_val[static_cast<int64_t>(b) * k + i] = ok ? xs[i] : 0.0;
  }
}

}  // namespace gift

using namespace gift;

extern "C" int gift_act_from_topk(const int32_t* topk_idx, const double* topk_val, int32_t B,
                                  int32_t kk, int32_t k1, int32_t cap, int32_t* act_idx,
                                  double* act_val, int32_t* act_cnt, double* act_norm,
                                  void* stream) {
  GIFT_REQUIRE(k1 >= 1, GIFT_ERR_INVALID, "k1 must be >= 1");
  GIFT_REQUIRE(cap >= min(k1, kk), GIFT_ERR_CAPACITY, "activation capacity too small");
  if (B <= 0) return GIFT_OK;
  act_from_topk_kernel<<<static_cast<unsigned>(cdiv(B, 4)), 128, 0, as_stream(stream)>>>(
      topk_idx, topk_val, B, kk, k1, cap, act_idx, act_val, act_cnt, act_norm);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_act_mean(const int32_t* raw_idx, const double* raw_val, const int32_t* raw_cnt,
                             int32_t raw_cap, const int32_t* nbr, int32_t B, int32_t k2,
                             int32_t cap, int32_t* out_idx, double* out_val, int32_t* out_cnt,
                             double* out_norm, void* stream) {
  GIFT_REQUIRE(k2 >= 0 && k2 <= MAX_NBR, GIFT_ERR_UNSUPPORTED, "k2 = %d > %d", k2, MAX_NBR);
  GIFT_REQUIRE(cap >= raw_cap * k2, GIFT_ERR_CAPACITY, "activation capacity too small");
  GIFT_REQUIRE(raw_cap * k2 <= AM_MAX_E, GIFT_ERR_UNSUPPORTED, "k1 * k2 = %d > %d",
               raw_cap * k2, AM_MAX_E);
  if (B <= 0) return GIFT_OK;
  act_mean_kernel<<<static_cast<unsigned>(cdiv(B, AM_WARPS)), AM_WARPS * 32, 0,
                    as_stream(stream)>>>(
      raw_idx, raw_val, raw_cnt, raw_cap, nbr, B, k2, cap, out_idx, out_val, out_cnt, out_norm);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_act_aggregate(const int32_t* a_idx, const double* a_val, const int32_t* a_cnt,
                                  int32_t a_cap, const int32_t* b_idx, const double* b_val,
                                  const int32_t* b_cnt, int32_t b_cap, int32_t B, double alpha,
                                  int32_t cap, int32_t* out_idx, double* out_val, int32_t* out_cnt,
                                  double* out_norm, void* stream) {
  GIFT_REQUIRE(alpha > 0.0, GIFT_ERR_INVALID, "alpha must be > 0");
  GIFT_REQUIRE(cap >= a_cap + b_cap, GIFT_ERR_CAPACITY, "aggregate capacity must be >= a_cap + b_cap");
  if (B <= 0) return GIFT_OK;
  act_aggregate_kernel<<<static_cast<unsigned>(cdiv(B, 128)), 128, 0, as_stream(stream)>>>(
      a_idx, a_val, a_cnt, a_cap, b_idx, b_val, b_cnt, b_cap, B, alpha, cap, out_idx, out_val,
      out_cnt, out_norm);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_act_compact(const int32_t* act_idx, const double* act_val,
                                const int32_t* act_cnt, int32_t cap, int64_t nrows,
                                int64_t* row_off, uint32_t* out_key, uint32_t* out_pos,
                                int32_t* out_owner, double* out_val, void* ws, size_t ws_bytes,
                                void* stream) {
  cudaStream_t st = as_stream(stream);
  int rc = scan_exclusive_i32_to_i64(act_cnt, row_off, nrows, true, ws, ws_bytes, st);
  if (rc != GIFT_OK) return rc;
  if (nrows <= 0 || out_key == nullptr) return GIFT_OK;
  act_compact_kernel<<<static_cast<unsigned>(cdiv(nrows, 128)), 128, 0, st>>>(
      act_idx, act_val, act_cnt, cap, nrows, row_off, out_key, out_pos, out_owner, out_val);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_sif_permute(const uint32_t* pos, const int32_t* owner, const double* val,
                                int64_t nnz, int32_t* e_ord, double* e_val, void* stream) {
  if (nnz <= 0) return GIFT_OK;
  sif_permute_kernel<<<static_cast<unsigned>(cdiv(nnz, 256)), 256, 0, as_stream(stream)>>>(
      pos, owner, val, nnz, e_ord, e_val);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

extern "C" int gift_sif_query(const int64_t* e_off, const int32_t* e_ord, const double* e_val,
                              const double* norms, int64_t n_global, int64_t n_local,
                              const int32_t* q_idx, const double* q_val, const int32_t* q_cnt,
                              const double* q_norm, int32_t B, int32_t cap, double* out_scores,
                              void* stream) {
  if (B <= 0 || n_local <= 0) return GIFT_OK;
  sif_query_kernel<<<static_cast<unsigned>(B), 256, 0, as_stream(stream)>>>(
      e_off, e_ord, e_val, norms, n_global, n_local, q_idx, q_val, q_cnt, q_norm, cap, out_scores);
  GIFT_LAUNCH_CHECK();
  return GIFT_OK;
}

// S-IF query implementations.  Big batches (B x max_touched >= 2^24 pairs
// bound: config 5) take the bucketed path (no host synchronisation), or the
// radix-sort one where the bucketed limits are exceeded; small batches the
// accumulator-row kernel.  flags GIFT_SIF_ROWS / SORT / BUCKET override.
enum SifMode { SIF_MODE_ROWS, SIF_MODE_SORT, SIF_MODE_BUCKET };

static int sif_bucket_rb(int64_t n_local) {
  int rb = SB_MIN_RB;
  while ((static_cast<int64_t>(SB_MAX_R) << rb) < n_local) ++rb;
  return rb;
}

static bool sif_bucket_ok(int32_t cap, int64_t max_touched, int64_t n_local) {
  if (cap > SB_MAX_E || max_touched >= (1LL << 31)) return false;
  const int rb = sif_bucket_rb(n_local);
  return rb <= SB_MAX_RB &&
         sif_split_smem(cap, static_cast<int>(cdiv(n_local, 1LL << rb))) <= 200 * 1024;
}

// The sort-based path sizes its pair buffers for B x max_touched (44 B per
// pair plus radix scratch); past 2^26 pairs (~3 GB) a hub-skewed bound would
// reserve far more than the real touch count needs, so those batches take the
// accumulator-row kernel instead (by default; GIFT_SIF_SORT still forces it).
constexpr int64_t SORT_MAX_PAIRS = 1LL << 26;

static bool sif_sort_ok(int64_t B, int64_t n_local) {
  int bbits = 1, jbits = 1;
  while ((1LL << bbits) < B) ++bbits;
  while ((1LL << jbits) < n_local) ++jbits;
  return bbits + jbits <= 32;  // (query, shape) keys must fit 32 bits
}

static SifMode sif_mode(int64_t B, int32_t cap, int64_t max_touched, int64_t n_local,
                        int32_t flags) {
  if (flags & GIFT_SIF_ROWS) return SIF_MODE_ROWS;
  if ((flags & GIFT_SIF_BUCKET) && sif_bucket_ok(cap, max_touched, n_local))
    return SIF_MODE_BUCKET;
  if ((flags & GIFT_SIF_SORT) && sif_sort_ok(B, n_local)) return SIF_MODE_SORT;
  if (flags) return SIF_MODE_ROWS;  // a forced mode outside its limits
  if (B * max_touched < (1LL << 24)) return SIF_MODE_ROWS;
  if (sif_bucket_ok(cap, max_touched, n_local)) return SIF_MODE_BUCKET;
  return (sif_sort_ok(B, n_local) && B * max_touched <= SORT_MAX_PAIRS) ? SIF_MODE_SORT
                                                                     : SIF_MODE_ROWS;
}

extern "C" int gift_sif_query_topk(const int64_t* e_off, const int32_t* e_ord, const double* e_val,
                                   const double* norms, int64_t n_global, int64_t n_local,
                                   const int32_t* q_idx, const double* q_val,
                                   const int32_t* q_cnt, const double* q_norm, int32_t B,
                                   int32_t cap, double* acc_rows, int32_t n_acc_rows,
                                   int64_t acc_stride, const int32_t* order,
                                   const int32_t* idrank,
                                   const int32_t* self_local, int64_t ord_base, int32_t k,
                                   int64_t max_touched, int32_t* out_idx, double* out_val,
                                   void* ws, size_t ws_bytes, int32_t flags, void* stream) {
  cudaStream_t st = as_stream(stream);
  GIFT_REQUIRE((flags & ~(GIFT_SIF_ROWS | GIFT_SIF_SORT | GIFT_SIF_BUCKET)) == 0 &&
                   __builtin_popcount(static_cast<unsigned>(flags)) <= 1,
               GIFT_ERR_INVALID, "bad S-IF query flags 0x%x", flags);
  GIFT_REQUIRE(k >= 1 && k <= 256, GIFT_ERR_UNSUPPORTED, "k = %d outside [1, 256]", k);
  GIFT_REQUIRE(n_acc_rows >= 1 && acc_rows != nullptr && order != nullptr, GIFT_ERR_INVALID,
               "sparse S-IF query needs accumulator rows and the id-rank order");
  GIFT_REQUIRE(acc_stride >= n_local, GIFT_ERR_INVALID, "accumulator row stride < n_local");
  if (B <= 0 || n_local <= 0) return GIFT_OK;
  const int64_t m = min64(max_touched, n_local) + k + 1;
  Arena ar(ws, ws_bytes);
  double* cs = ar.take<double>(static_cast<int64_t>(B) * m);
  uint32_t* ct = ar.take<uint32_t>(static_cast<int64_t>(B) * m);
  int32_t* ci = ar.take<int32_t>(static_cast<int64_t>(B) * m);
  int32_t* cnt = ar.take<int32_t>(B);
  GIFT_REQUIRE(cs && ct && ci && cnt, GIFT_ERR_CAPACITY, "sparse S-IF workspace too small");
  int bbits = 1, jbits = 1;
  while ((1LL << bbits) < B) ++bbits;
  while ((1LL << jbits) < n_local) ++jbits;
  const SifMode mode = sif_mode(B, cap, max_touched, n_local, flags);
  if (mode == SIF_MODE_BUCKET) {
    const int rb = sif_bucket_rb(n_local);
    const int R = static_cast<int>(cdiv(n_local, 1LL << rb));
    const int64_t tmax = static_cast<int64_t>(B) * max_touched;
    const int64_t nc = tmax + static_cast<int64_t>(B) * (k + 1);
    Arena ab(ws, ws_bytes);
    double* bcs = ab.take<double>(nc);
    uint32_t* bct = ab.take<uint32_t>(nc);
    int32_t* bci = ab.take<int32_t>(nc);
    int32_t* tcnt = ab.take<int32_t>(B);
    int64_t* off = ab.take<int64_t>(B + 1);
    int32_t* bst = ab.take<int32_t>(static_cast<int64_t>(B) * (R + 1));
    int32_t* ntb = ab.take<int32_t>(static_cast<int64_t>(B) * R);
    uint16_t* pj = ab.take<uint16_t>(tmax);
    double* pc = ab.take<double>(tmax);
    const size_t sws = scan_ws_bytes(B);
    GIFT_REQUIRE(bcs && bct && bci && tcnt && off && bst && ntb && pj && pc &&
                     ab.remaining() >= sws + 256,
                 GIFT_ERR_CAPACITY, "bucketed S-IF workspace too small");
    sif_tcount_kernel<<<static_cast<unsigned>(cdiv(B, 8)), 256, 0, st>>>(q_idx, q_cnt, cap, e_off,
                                                                       n_global, B, tcnt);
    GIFT_LAUNCH_CHECK();
    int rc = scan_exclusive_i32_to_i64(tcnt, off, B, true, ab.base + align_up(ab.used, 256), sws,
                                       st);
    if (rc) return rc;
    const size_t ssm = sif_split_smem(cap, R);
    GIFT_CUDA_TRY(cudaFuncSetAttribute(sif_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(ssm)));
    sif_split_kernel<<<static_cast<unsigned>(min64(B, sm_count())), SB_WARPS * 32, ssm, st>>>(
        q_idx, q_val, q_cnt, cap, B, e_off, e_ord, e_val, n_global, rb, R, off, bst, pj, pc);
    GIFT_LAUNCH_CHECK();
    const int W = 1 << rb;
    const int rw =
        static_cast<int>(min64(16, (SB_RED_KB * 1024) / (static_cast<int64_t>(W) * 8)));
    const size_t rsm = static_cast<size_t>(rw) * W * 8;
    GIFT_CUDA_TRY(cudaFuncSetAttribute(sif_bucket_reduce_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(rsm)));
    const int64_t grid =
        min64(static_cast<int64_t>(sm_count()) * SB_RED_CTAS, cdiv(static_cast<int64_t>(B) * R, rw * 4));
    sif_bucket_reduce_kernel<<<static_cast<unsigned>(grid), rw * 32, rsm, st>>>(pj, pc, off, bst, B,
                                                                               R, rb, ntb);
    GIFT_LAUNCH_CHECK();
    const size_t ksm = sif_rank_smem(R);
    GIFT_CUDA_TRY(cudaFuncSetAttribute(sif_bucket_rank_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(ksm)));
    sif_bucket_rank_kernel<<<static_cast<unsigned>(B), RK_THREADS, ksm, st>>>(
        pj, pc, off, bst, ntb, R, rb, norms, q_norm, order, idrank, self_local, ord_base, n_local, k,
        bcs, bct, bci, out_idx, out_val);
    GIFT_LAUNCH_CHECK();
    return GIFT_OK;
  }
  if (mode == SIF_MODE_ROWS) {
    const int grid = min(B, n_acc_rows);
    sif_query_sparse_kernel<<<static_cast<unsigned>(grid), 256, 0, st>>>(
        e_off, e_ord, e_val, norms, n_global, n_local, q_idx, q_val, q_cnt, q_norm, B, cap,
        acc_rows, acc_stride, order, idrank, self_local, ord_base, k, m, cs, ct, ci, cnt);
    GIFT_LAUNCH_CHECK();
    return topk_rows_from_lists(cs, ct, ci, cnt, B, m, k, 0, out_idx, out_val, st);
  }
  // sort-based path: pairs emitted per query, radix-sorted by (b, j), runs summed
  int32_t* tcnt = ar.take<int32_t>(B);
  int64_t* off = ar.take<int64_t>(B + 1);
  const int64_t tmax = static_cast<int64_t>(B) * max_touched;
  uint32_t* keys = ar.take<uint32_t>(tmax);
  uint32_t* vals = ar.take<uint32_t>(tmax);
  double* contrib = ar.take<double>(tmax);
  int32_t* rflag = ar.take<int32_t>(tmax);
  int64_t* rpos = ar.take<int64_t>(tmax + 1);
  GIFT_REQUIRE(tcnt && off && keys && vals && contrib && rflag && rpos, GIFT_ERR_CAPACITY,
               "sparse S-IF workspace too small");
  sif_tcount_kernel<<<static_cast<unsigned>(cdiv(B, 8)), 256, 0, st>>>(q_idx, q_cnt, cap, e_off,
                                                                     n_global, B, tcnt);
  GIFT_LAUNCH_CHECK();
  const size_t sws = scan_ws_bytes(B);
  void* scan_ws = ar.base + align_up(ar.used, 256);
  GIFT_REQUIRE(ar.remaining() >= sws + 256, GIFT_ERR_CAPACITY, "sparse S-IF workspace too small");
  int rc = scan_exclusive_i32_to_i64(tcnt, off, B, true, scan_ws, sws, st);
  if (rc) return rc;
  int64_t T = 0;
  GIFT_CUDA_TRY(cudaMemcpyAsync(&T, off + B, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA_TRY(cudaStreamSynchronize(st));
  GIFT_REQUIRE(T <= tmax, GIFT_ERR_CAPACITY, "sparse S-IF workspace too small");
  sif_emit_kernel<<<static_cast<unsigned>(B), 256, 0, st>>>(q_idx, q_val, q_cnt, cap, e_off, e_ord,
                                                           e_val, n_global, jbits, off, keys, vals,
                                                           contrib);
  GIFT_LAUNCH_CHECK();
  if (T > 0) {
    uint32_t* ktmp = ar.take<uint32_t>(tmax);
    uint32_t* vtmp = ar.take<uint32_t>(tmax);
    GIFT_REQUIRE(ktmp && vtmp && ar.remaining() > 256, GIFT_ERR_CAPACITY,
                 "sparse S-IF workspace too small");
    void* rws = ar.base + align_up(ar.used, 256);
    rc = gift_radix_sort_pairs(keys, vals, T, bbits + jbits, ktmp, vtmp, rws,
                               ar.remaining() - 256, st);
    if (rc) return rc;
    double* csorted = ar.take<double>(tmax);
    GIFT_REQUIRE(csorted != nullptr && ar.remaining() > 256, GIFT_ERR_CAPACITY,
                 "sparse S-IF workspace too small");
    sif_runflag_kernel<<<static_cast<unsigned>(cdiv(T, 256)), 256, 0, st>>>(keys, vals, contrib, T,
                                                                          rflag, csorted);
    GIFT_LAUNCH_CHECK();
    rc = scan_exclusive_i32_to_i64(rflag, rpos, T, true, ar.base + align_up(ar.used, 256),
                                   ar.remaining() - 256, st);
    if (rc) return rc;
    sif_runsum_kernel<<<static_cast<unsigned>(cdiv(T, 256)), 256, 0, st>>>(
        keys, vals, csorted, T, jbits, off, rpos, norms, q_norm, idrank, self_local, ord_base, m,
        cs, ct, ci);
    GIFT_LAUNCH_CHECK();
  } else {
    GIFT_CUDA_TRY(cudaMemsetAsync(rpos, 0, sizeof(int64_t), st));
  }
  sif_fill_kernel<<<static_cast<unsigned>(cdiv(B, 8)), 256, 0, st>>>(
      keys, off, rpos, jbits, order, idrank, self_local, ord_base, n_local, k, B, m, cs, ct, ci,
      cnt);
  GIFT_LAUNCH_CHECK();
  return topk_rows_from_lists(cs, ct, ci, cnt, B, m, k, 0, out_idx, out_val, st);
}

extern "C" size_t gift_sif_query_topk_ws_bytes(int32_t B, int32_t cap, int64_t n_local, int32_t k,
                                               int64_t max_touched, int32_t flags) {
  const int64_t m = min64(max_touched, n_local) + k + 1;
  size_t bytes = static_cast<size_t>(B) * m * 16 + static_cast<size_t>(B) * 4 + 4096;
  const SifMode mode = sif_mode(B, cap, max_touched, n_local, flags);
  if (mode == SIF_MODE_BUCKET) {  // candidates, pairs, bucket starts
    const int64_t tmax = static_cast<int64_t>(B) * max_touched;
    const int64_t R = cdiv(n_local, 1LL << sif_bucket_rb(n_local));
    const int64_t nc = tmax + static_cast<int64_t>(B) * (k + 1);
    return static_cast<size_t>(nc) * 16 + static_cast<size_t>(tmax) * 10 +
           static_cast<size_t>(B) * (4 + 8 + 4 * (2 * R + 1)) + scan_ws_bytes(B) + 16 * 256 + 4096;
  }
  if (mode == SIF_MODE_SORT) {  // sort-based path: pairs + radix scratch
    const int64_t tmax = static_cast<int64_t>(B) * max_touched;
    bytes += static_cast<size_t>(B) * 12 + 1024 + static_cast<size_t>(tmax) * 44 + 8 +
             scan_ws_bytes(B) + scan_ws_bytes(tmax) + gift_radix_sort_ws_bytes(tmax) + 8192;
  }
  return bytes;
}
