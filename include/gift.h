/*
 * gift.h — C ABI of the B200-native GIFT query path (libgift.so).
 *
 * The reference (`/root/reference/pkg`, package `shapesearch`) is pure Python +
 * numpy and has no FFI layer of its own; its boundary is the Python API in
 * `shapesearch/index.py` and the module functions it composes.  Every entry
 * point below replaces one numpy call site of that path and names the
 * reference function (file:line) whose semantics it reproduces.  The Python
 * binding a maintainer would add is shown in INTEGRATION.md (ctypes).
 *
 * Conventions
 *   - plain pointers and sizes only; all array pointers are DEVICE pointers
 *     unless stated otherwise; all buffers are caller-allocated (the library
 *     never allocates or frees caller memory);
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on that stream unless stated otherwise;
 *   - every call returns GIFT_OK (0) or an error code; the message of the last
 *     error on the calling thread is available from gift_last_error();
 *   - dtype codes: GIFT_F32 = 0, GIFT_F16 = 1, GIFT_F64 = 2.
 *   - entry points are reentrant given distinct outputs, workspaces and
 *     streams; there is no hidden global mutable state besides the
 *     thread-local error message.
 */
#ifndef GIFT_H_
#define GIFT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped onto shapesearch.errors by the Python shim) ---- */
#define GIFT_OK 0
#define GIFT_ERR_INVALID 1     /* ValueError                                  */
#define GIFT_ERR_DIM 2         /* errors.DimensionMismatch  (errors.py:28)    */
#define GIFT_ERR_EMPTY 3       /* errors.EmptySet           (errors.py:36)    */
#define GIFT_ERR_CUDA 4        /* CUDA runtime failure                        */
#define GIFT_ERR_CAPACITY 5    /* workspace too small (size reported)         */
#define GIFT_ERR_UNSUPPORTED 6 /* shape outside the kernels' supported range  */

#define GIFT_F32 0
#define GIFT_F16 1
#define GIFT_F64 2

#define GIFT_SIM_COSINE 0   /* clip(q.p, 0, 1)          matching.py:158      */
#define GIFT_SIM_GAUSSIAN 1 /* exp(-|q-p|^2 / sigma^2)   north_star (D1)      */

/* Device-resident first inverted file of one shard (cell-major CSR).
 * Replaces matching.FirstInvertedFile (matching.py:64-103).  Built by the
 * gift_fif_* build calls below; all pointers are device pointers. */
#define GIFT_FIF_TILED_SEGMENTS 1
/* flags bits 8-15: SMs the F-IF scan leaves to the kernels of other query
 * batches in flight on other streams (0: one persistent scan CTA per SM) */
#define GIFT_FIF_RESERVE_SMS(n) (((n) & 255) << 8)
/* Kernel variants (all bit-identical or within the same 1e-5 contract; the
 * defaults are the measured-fastest per index).  Selected by
 * the caller through the view -- the library reads no environment.        */
#define GIFT_FIF_SCAN_SIMT (1 << 16)   /* CUDA-core scan instead of tcgen05   */
#define GIFT_FIF_QUANT_SIMT (1 << 17)  /* CUDA-core quantize stage 1          */
#define GIFT_FIF_REDUCE_SHIFT 18       /* bits 18-19: view-best reduce:       */
#define GIFT_FIF_REDUCE_AUTO 0         /*   by shard size (owner >= 32k)      */
#define GIFT_FIF_REDUCE_RANGE 1
#define GIFT_FIF_REDUCE_GATHER 2
#define GIFT_FIF_REDUCE_OWNER 3
#define GIFT_FIF_REDUCE(m) (((m) & 3) << GIFT_FIF_REDUCE_SHIFT)
#define GIFT_FIF_SCHED_STATIC (1 << 20) /* static CTA stride over scan items   */
#define GIFT_FIF_PAIR_SHIFT 21          /* bits 21-22: cta_group::2 scan:      */
#define GIFT_FIF_PAIR_AUTO 0            /*   pairs iff the f32 lo plane exists */
#define GIFT_FIF_PAIR_OFF 1
#define GIFT_FIF_PAIR_ON 2
#define GIFT_FIF_PAIR(m) (((m) & 3) << GIFT_FIF_PAIR_SHIFT)
#define GIFT_FIF_DRAIN_SHIFT 24         /* bits 24-28: D1 drain interval in    */
#define GIFT_FIF_DRAIN_KB(n) (((n) & 31) << GIFT_FIF_DRAIN_SHIFT) /* 64-wide */
                                        /* k-blocks, 1..16 (0 = the default:   */
                                        /* 8: max 2.1e-6 vs the 1e-5 contract) */
#define GIFT_FIF_RAW_ACCUM (1 << 29)    /* no truncation compensation of the   */
                                        /* tensor-core accumulators (tests)    */
#define GIFT_FIF_DENSE_OFF (1 << 30)    /* fp16 storage: no probe-major pair   */
                                        /* scan of the cells with >= 192       */
                                        /* probes (fif_scan_dense.cu)          */

typedef struct gift_fif_view {
  int32_t K;                 /* codebook size                                 */
  int32_t d;                 /* feature dimension                             */
  int32_t dtype;             /* storage dtype of feat: GIFT_F32 / GIFT_F16    */
  int32_t flags;             /* GIFT_FIF_TILED_SEGMENTS: no segment is longer   */
                             /* than a scan tile (every compact entry is       */
                             /* written once; no zero-fill needed);            */
                             /* GIFT_FIF_RESERVE_SMS(n); kernel variants below */
  int64_t n_postings;        /* P                                             */
  int64_t n_segments;        /* S: (cell, shape) runs                          */
  int64_t n_tiles;           /* T: scan tiles (whole segments, <= tile_n)     */
  int64_t n_local;           /* shapes owned by this shard                    */
  int64_t ord_base;          /* first global ordinal of this shard            */
  const int64_t* cell_off;   /* [K+1] posting offsets per cell                */
  const int32_t* post_ord;   /* [P] global shape ordinal per posting          */
  const void* feat;          /* [P, d] stored view features, cell-major       */
  const float* pnorm2;       /* [P] |p|^2 (gaussian mode)                     */
  const int64_t* seg_off;    /* [K+1] segment offsets per cell                */
  const int32_t* seg_ord;    /* [S] shape ordinal of each segment             */
  const int32_t* seg_pstart; /* [S+1] first posting of each segment           */
  const int64_t* tile_off;   /* [K+1] tile offsets per cell                   */
  const int32_t* tile_pstart;/* [T]                                           */
  const int32_t* tile_pend;  /* [T]                                           */
  const int32_t* tile_seg0;  /* [T] first segment overlapping the tile        */
  const int32_t* tile_seg1;  /* [T] one past the last                         */
  const float* centroids;    /* [K, d] f32 codebook (codebook.py:22-34)       */
  const double* cnorm2;      /* [K] |c|^2 in f64                              */
  double cmax_norm;          /* max_c |c|                                     */
  const void* feat_hi;       /* [P, d] fp16 plane h1 = rn(feat) (tensor-core  */
  const void* feat_lo;       /* scan); feat_lo: rn((feat-h1) 2^11), NULL for   */
                             /* fp16 storage (feat_hi == feat)                 */
  /* shape -> segment map (optional; NULL selects the per-range reduce):      */
  const int64_t* shape_seg_off; /* [n_local+1] segments of each local shape   */
  const int32_t* shape_seg;     /* [S] global segment index, ascending cell   */
  const int32_t* shape_seg_cell;/* [S] cell of segment shape_seg[g]           */
  int64_t max_cell_segments;    /* max over cells of its segment count         */
  const uint8_t* seg_single;    /* [S] 1: the segment's shape has no other    */
                                /* segment (all its views in one cell; the    */
                                /* owner reduce skips its shape lookups);     */
                                /* optional (NULL)                            */
} gift_fif_view;

/* ---- library ---- */
int gift_version(void);
int gift_last_error(char* buf, size_t len);
int gift_fif_tile_n(void); /* posting-tile height of the scan kernel */

/* ---- K1 quantize: replaces codebook.quantize (codebook.py:111-124) ----
 * For each of n vectors X[i] (dtype f32/f16/f64, row-major [n, d]) writes the
 * ma nearest centroids, ascending by the reference's f64 direct-difference
 * squared distance (numpy pairwise summation order), ties to the lower index.
 * Bit-exact with the reference.  If nz != NULL, rows with nz[i] == 0 get
 * out_idx = -1 (query_fif skips zero views, matching.py:150-151); if
 * zero_key >= 0 such rows get zero_key instead (F-IF build sort key).
 * Workspace: at least gift_quantize_ws_bytes(128, d, K, xdtype); larger
 * workspaces process more rows per pass. */
size_t gift_quantize_ws_bytes(int64_t n, int32_t d, int32_t K, int32_t xdtype);
int gift_quantize(const void* X, int32_t xdtype, int64_t n, int32_t d,
                  const float* C, const double* cnorm2, int32_t K,
                  double cmax_norm, int32_t ma, const uint8_t* nz,
                  int32_t zero_key, int32_t* out_idx, void* ws,
                  size_t ws_bytes, void* stream);
/* gift_quantize with explicit stage-1 selection: flags = 0 (tensor cores
 * when d % 8 == 0) or GIFT_QUANT_SIMT (CUDA cores); same results. */
#define GIFT_QUANT_SIMT 1
int gift_quantize_ex(const void* X, int32_t xdtype, int64_t n, int32_t d,
                     const float* C, const double* cnorm2, int32_t K,
                     double cmax_norm, int32_t ma, const uint8_t* nz,
                     int32_t zero_key, int32_t* out_idx, void* ws,
                     size_t ws_bytes, int32_t flags, void* stream);

/* GIFTFT1 ingest: out[r, :] = f32(x[r, :] / norms[r]) (IEEE f64 division),
 * rows with norms[r] == 0 copied unchanged -- features.py:67-71 `_unit`, the
 * per-row re-normalization of import_features (features.py:140-185); norms
 * are the host's f64 sqrt(x.dot(x)).  x and out may alias. */
int gift_normalize_rows(const float* x, const double* norms, int64_t rows, int32_t d,
                        float* out, void* stream);

/* ---- codebook training (codebook.py:37-108, train_codebook) ----------------
 * Device half of k-means++ and Lloyd's iterations in f64; the host runs the
 * reference's control flow and numpy RNG stream.
 * gift_rows_sqnorm_f64: out[r] = sum_j X[r,j]^2 in numpy's pairwise order
 *   ((points * points).sum(axis=1), codebook.py:39-41).
 * gift_kmeans_assign: per point the nearest center by
 *   max((|x|^2 - 2 x.c) + |c|^2, 0) (codebook.py:37-45), ties to the lower
 *   index (argmin, codebook.py:84-85); out_label / out_mind2 may be NULL.
 * gift_kmeans_update: out[c,:] = (sum of X[order[m],:] for m in
 *   [off[c], off[c+1]) in that order, from 0.0) / (off[c+1] - off[c])
 *   (np.add.at + division, codebook.py:96-98); order = points stably sorted
 *   by label. */
int gift_rows_sqnorm_f64(const double* X, int64_t n, int32_t d, double* out, void* stream);
int gift_kmeans_assign(const double* X, int64_t n, int32_t d, const double* C, int32_t k,
                       const double* xn2, const double* cn2, int32_t* out_label,
                       double* out_mind2, void* stream);
int gift_kmeans_update(const double* X, int64_t n, int32_t d, const int64_t* order,
                       const int64_t* off, int32_t k, double* out_centers, void* stream);

/* Per-view non-zero flag and |x|^2 (f64 accumulate, stored f32).
 * `row.any()` tests of matching.py:121 / :150. */
int gift_view_prep(const void* X, int32_t xdtype, int64_t nviews, int32_t d,
                   uint8_t* out_nz, float* out_norm2, void* stream);

/* ---- K2 support: stable LSD radix sort of (u32 key, u32 value) pairs ----
 * Sorted result is left in keys/vals.  Stable: equal keys keep input order
 * (the reference appends postings in shape-major, view-minor order,
 * matching.py:112-125, and activations in owner order, rerank.py:194-198). */
size_t gift_radix_sort_ws_bytes(int64_t n);
int gift_radix_sort_pairs(uint32_t* keys, uint32_t* vals, int64_t n,
                          int32_t key_bits, uint32_t* keys_tmp,
                          uint32_t* vals_tmp, void* ws, size_t ws_bytes,
                          void* stream);
/* out_off[b] = first position of key b in a sorted key array, b in [0, nb]. */
int gift_offsets_from_sorted(const uint32_t* keys, int64_t n, int64_t nbuckets,
                             int64_t* out_off, void* stream);

/* ---- K2 F-IF build: replaces matching.build_fif (matching.py:106-133) ----
 * gather: out_feat[p] = src[perm[p]] (rows of d), out_ord[p] = ord_base +
 * perm[p] / V, out_pnorm2[p] = |src[perm[p]]|^2. */
int gift_fif_gather(const void* src, int32_t dtype, int32_t d, int32_t V,
                    const uint32_t* perm, int64_t P, int64_t ord_base,
                    void* out_feat, int32_t* out_ord, float* out_pnorm2,
                    void* stream);
/* Streamed build (database larger than what fits twice in HBM; the
 * reference's build_fif, matching.py:106-133, over chunks of shapes):
 * pass 1 quantizes chunk by chunk into one key per view and radix-sorts them
 * (perm = cell-major view order); gift_perm_invert gives every view its
 * posting (pos[view] = p, -1 for zero views); pass 2 calls gift_fif_scatter
 * per chunk: rows of the chunk's views (global views view_base..) land at
 * their postings in out_feat (storage dtype, may be NULL) and/or the
 * tensor-core planes out_hi/out_lo (fp16, x = hi + 2^-11 lo; f16 storage
 * needs only out_hi), with out_ord / out_pnorm2 exactly as gift_fif_gather. */
int gift_perm_invert(const uint32_t* perm, int64_t P, int64_t n_total,
                     int32_t* pos, void* stream);
int gift_fif_scatter(const void* src, int32_t dtype, int32_t d, int32_t V,
                     int64_t n_views, const int32_t* pos, int64_t view_base,
                     int64_t ord_base, void* out_feat, void* out_hi,
                     void* out_lo, int32_t* out_ord, float* out_pnorm2,
                     void* stream);
/* Segments = maximal runs of one shape inside one cell.  Two passes: with
 * seg_ord == NULL only seg_off[K+1] is written (read seg_off[K] = S), then
 * call again with seg_ord/seg_pstart allocated ([S], [S+1]). */
size_t gift_fif_build_ws_bytes(int64_t P, int32_t K);
int gift_fif_segments(const int64_t* cell_off, const int32_t* post_ord,
                      int32_t K, int64_t P, int64_t* seg_off, int32_t* seg_ord,
                      int32_t* seg_pstart, void* ws, size_t ws_bytes,
                      void* stream);
/* Scan tiles: greedy packing of whole segments into tiles of <= tile_n
 * postings (segments longer than tile_n are split).  Two passes as above. */
int gift_fif_tiles(const int64_t* cell_off, const int64_t* seg_off,
                   const int32_t* seg_pstart, int32_t K, int32_t tile_n,
                   int64_t* tile_off, int32_t* tile_pstart, int32_t* tile_pend,
                   int32_t* tile_seg0, int32_t* tile_seg1, void* ws,
                   size_t ws_bytes, void* stream);
/* Tensor-core operand planes of f32 rows: h1 = rn16(x), h2 = rn16((x - h1)
 * 2^11), so x = h1 + 2^-11 h2 to 22 significant bits (fif_scan_tc.cu). */
int gift_split_planes(const float* x, int64_t n, void* h1, void* h2,
                      void* stream);
/* out[i] = src[idx[i]] widened to f32 (query_by_id's shape_matrix,
 * matching.py:94-103, index.py:302-314). */
int gift_gather_rows_f32(const void* src, int32_t dtype, int32_t d,
                         const int64_t* idx, int64_t n, float* out,
                         void* stream);
/* Same from the tensor-core planes of an index that keeps no storage copy
 * (streamed config-3 build): out = hi + 2^-11 lo (22 significant bits). */
int gift_gather_rows_planes(const void* hi, const void* lo, int32_t d,
                            const int64_t* idx, int64_t n, float* out,
                            void* stream);

/* ---- K3 F-IF score: replaces matching.query_fif (matching.py:136-161) ----
 * Batched: Q is [B*V, d] f32 (B queries of V views).  Writes dense f64
 * scores [B, n_local] for the shard's shapes: mean over the query's views of
 * the best similarity among postings of the view's ma nearest cells; never
 * visited shapes score exactly 0.  vq (nullable) overrides the per-query
 * divisor (default V).  Workspace layout is internal; the first 64 bytes hold
 * int64 status words: [0] work items, [1] compact outputs needed,
 * [2] overflow flag (1 = workspace too small: grow to
 * gift_fif_score_ws_bytes(.., needed) and rerun). */
size_t gift_fif_score_ws_bytes(const gift_fif_view* f, int32_t B, int32_t V,
                               int32_t ma, int64_t compact_capacity);
int gift_fif_score(const gift_fif_view* f, const float* Q, int32_t B,
                   int32_t V, const int32_t* vq, int32_t ma, int32_t mode,
                   double sigma, double* out_scores, void* ws,
                   size_t ws_bytes, void* stream);
/* Same, recording the caller's cudaEvent_t handles (nullable) on `stream`
 * immediately before and after the scan kernel (bench roofline timing). */
int gift_fif_score_ex(const gift_fif_view* f, const float* Q, int32_t B,
                      int32_t V, const int32_t* vq, int32_t ma, int32_t mode,
                      double sigma, double* out_scores, void* ws,
                      size_t ws_bytes, void* stream, void* ev_scan_begin,
                      void* ev_scan_end);

/* Same, and with cand_k in [1, 8] also the best cand_k shapes (score desc,
 * ordinal asc; -1 padded) of every (query, shape range) of the reduce:
 * cand_s/cand_i [B][gift_fif_score_ranges2(f, V, ma)][cand_k] — merged by
 * gift_topk_cand into rerank.top_neighbors (rerank.py:78-87).  With
 * cand_k > 0, out_scores may be NULL (candidates only, no dense scores).
 * gift_fif_score_ranges is the ma-agnostic form (valid when the index has no
 * shape -> segment map). */
int gift_fif_score_ranges(const gift_fif_view* f, int32_t V);
int gift_fif_score_ranges2(const gift_fif_view* f, int32_t V, int32_t ma);
/* Reduce the score call will use: 0 per-range tiles, 1 gather, 2 owner. */
int gift_fif_reduce_mode(const gift_fif_view* f, int32_t V, int32_t ma);
int gift_fif_score_ex2(const gift_fif_view* f, const float* Q, int32_t B,
                       int32_t V, const int32_t* vq, int32_t ma, int32_t mode,
                       double sigma, double* out_scores, void* ws,
                       size_t ws_bytes, void* stream, void* ev_scan_begin,
                       void* ev_scan_end, int32_t cand_k, double* cand_s,
                       int32_t* cand_i);

/* ---- K4 top-k: replaces the lexsort selections rerank.py:74, :86-87 and
 * index.py:290-294.  Per row of a dense f64 score matrix [B, n], returns the
 * k best by (score desc, tiebreak asc) where tiebreak(j) = 0 if
 * j == self_local[b] else 1 + (idrank ? idrank[j] : ord_base + j).  Output
 * global ordinals (ord_base + j); with positive_only, entries scoring <= 0
 * are reported as -1.  k <= 2048. */
int gift_topk_rows(const double* scores, int32_t B, int64_t n, int32_t k,
                   const int32_t* idrank, const int32_t* self_local,
                   int64_t ord_base, int32_t positive_only, int32_t* out_idx,
                   double* out_val, void* stream);
/* Same, with a workspace of >= gift_topk_ws_bytes(B, n, k): rows are split
 * into slices scanned by separate CTAs, then merged (identical result). */
size_t gift_topk_ws_bytes(int32_t B, int64_t n, int32_t k);
int gift_topk_rows_ex(const double* scores, int32_t B, int64_t n, int32_t k,
                      const int32_t* idrank, const int32_t* self_local,
                      int64_t ord_base, int32_t positive_only,
                      int32_t* out_idx, double* out_val, void* ws,
                      size_t ws_bytes, void* stream);

/* Best k of m explicit candidates per row (cs scores, ci global ordinals,
 * -1 = none), key (score desc, ordinal asc); positive_only as above. */
int gift_topk_cand(const double* cs, const int32_t* ci, int32_t B, int64_t m,
                   int32_t k, int32_t positive_only, int32_t* out_idx,
                   double* out_val, void* stream);
/* gift_topk_cand with an explicit tiebreak per candidate (ct, uint32: the
 * key is (score desc, tiebreak asc)); candidates with ci < 0 are absent.
 * Merges the per-shard candidates of the sharded engine (one all-gather per
 * exchange): tiebreak = ordinal for the neighbour lists (rerank.py:86),
 * 0 (own entry) / 1 + id rank for the final ranking (index.py:290-294). */
int gift_topk_cand_tb(const double* cs, const int32_t* ci, const uint32_t* ct, int32_t B,
                      int64_t m, int32_t k, int32_t positive_only, int32_t* out_idx,
                      double* out_val, void* stream);

/* ---- K5 activations (fixed-capacity rows: idx[B,cap] asc, val, cnt, norm) */
/* build_activation (rerank.py:64-75) from a top-k result: first k1 positive
 * entries, re-sorted by ordinal, norm = sequential ascending sum. */
int gift_act_from_topk(const int32_t* topk_idx, const double* topk_val,
                       int32_t B, int32_t kk, int32_t k1, int32_t cap,
                       int32_t* act_idx, double* act_val, int32_t* act_cnt,
                       double* act_norm, void* stream);
/* mean_activation (rerank.py:90-100): out[b] = mean of raw[nbr[b, t]] over
 * the valid (>= 0) neighbours t, accumulated in neighbour order. */
int gift_act_mean(const int32_t* raw_idx, const double* raw_val,
                  const int32_t* raw_cnt, int32_t raw_cap, const int32_t* nbr,
                  int32_t B, int32_t k2, int32_t cap, int32_t* out_idx,
                  double* out_val, int32_t* out_cnt, double* out_norm,
                  void* stream);
/* aggregate (rerank.py:128-147): generalized mean over the union support. */
int gift_act_aggregate(const int32_t* a_idx, const double* a_val,
                       const int32_t* a_cnt, int32_t a_cap,
                       const int32_t* b_idx, const double* b_val,
                       const int32_t* b_cnt, int32_t b_cap, int32_t B,
                       double alpha, int32_t cap, int32_t* out_idx,
                       double* out_val, int32_t* out_cnt, double* out_norm,
                       void* stream);

/* ---- K5/K6 S-IF: replaces rerank.build_sif / query_sif (rerank.py:187-230)
 * compact: rows [0, nrows) of an activation matrix -> (key = coordinate,
 * value = position) pairs in row-major order plus owner/value per position;
 * row_off[nrows+1] is written (exclusive scan of cnt). */
int gift_act_compact(const int32_t* act_idx, const double* act_val,
                     const int32_t* act_cnt, int32_t cap, int64_t nrows,
                     int64_t* row_off, uint32_t* out_key, uint32_t* out_pos,
                     int32_t* out_owner, double* out_val, void* ws,
                     size_t ws_bytes, void* stream);
/* permute: e_ord[q] = owner[pos[q]], e_val[q] = val[pos[q]]. */
int gift_sif_permute(const uint32_t* pos, const int32_t* owner,
                     const double* val, int64_t nnz, int32_t* e_ord,
                     double* e_val, void* stream);
/* Dense re-ranked scores [B, n_local]: acc_j accumulates min(Fq[i], F_j[i])
 * over the query support in ascending i (f64, sequential per j), then
 * S' = acc / ((|Fq|_1 + |F_j|_1) - acc) on touched shapes, 0 elsewhere. */
int gift_sif_query(const int64_t* e_off, const int32_t* e_ord,
                   const double* e_val, const double* norms, int64_t n_global,
                   int64_t n_local, const int32_t* q_idx, const double* q_val,
                   const int32_t* q_cnt, const double* q_norm, int32_t B,
                   int32_t cap, double* out_scores, void* stream);

/* query_sif + the final ranking of index.query (index.py:290-294) without
 * dense rows: touched shapes only, plus the reference's zero-score fill (self
 * first, then id-rank order).  Returns the k best by (score desc, tiebreak
 * asc) exactly like gift_topk_rows over the dense scores.  acc_rows:
 * n_acc_rows rows of acc_stride (>= n_local) f64, all zero on entry and on
 * return (caller-owned scratch; a stride that is not a multiple of a large
 * power of two keeps the rows' hot entries on different DRAM channels).  order[r] = local shape of id rank r (inverse of idrank).
 * max_touched: an upper bound of the shapes one query can touch (support cap
 * x the longest S-IF entry). */
/* flags: 0 = by batch size (B x max_touched >= 2^24: the bucketed path, or
 * the sort-based one beyond the bucketed limits -- cap <= 1024 support
 * entries, n_local <= 2^24), GIFT_SIF_ROWS = per-query accumulator rows,
 * GIFT_SIF_SORT = (query, shape) pairs radix-sorted, GIFT_SIF_BUCKET = pairs
 * split by shape range and reduced in shared memory (no host
 * synchronisation).  All give identical results; a forced mode outside its
 * limits falls back to the rows path. */
#define GIFT_SIF_ROWS 1
#define GIFT_SIF_SORT 2
#define GIFT_SIF_BUCKET 4
size_t gift_sif_query_topk_ws_bytes(int32_t B, int32_t cap, int64_t n_local, int32_t k,
                                    int64_t max_touched, int32_t flags);
int gift_sif_query_topk(const int64_t* e_off, const int32_t* e_ord,
                        const double* e_val, const double* norms,
                        int64_t n_global, int64_t n_local, const int32_t* q_idx,
                        const double* q_val, const int32_t* q_cnt,
                        const double* q_norm, int32_t B, int32_t cap,
                        double* acc_rows, int32_t n_acc_rows,
                        int64_t acc_stride, const int32_t* order,
                        const int32_t* idrank,
                        const int32_t* self_local, int64_t ord_base, int32_t k,
                        int64_t max_touched, int32_t* out_idx, double* out_val,
                        void* ws, size_t ws_bytes, int32_t flags, void* stream);

/* ---- exact set matching: replaces matching.exact_hausdorff_distance and
 * matching.exact_similarity (matching.py:39-61).  For every (query set b,
 * target set n): out[(b N + n) 3 + 0] = robust Hausdorff mean_v(1 - max_u
 * q_v.p_u), [1] = standard max_v(1 - max_u q_v.p_u), [2] = exact similarity
 * mean_v clip(max_u q_v.p_u, 0, 1), dots in f64.  Q [B, Vq, d], P [N, Vp,
 * d] (dtype f32 or f64); q_cnt / p_cnt (optional) = views per set. */
int gift_exact_sets(const void* Q, int32_t qdtype, const int32_t* q_cnt, int32_t B,
                    int32_t Vq, const void* P, int32_t pdtype, const int32_t* p_cnt,
                    int32_t N, int32_t Vp, int32_t d, double* out, void* stream);

/* ---- query_fif in f64 (matching.py:136-161), the opt-in exact-precision
 * scan: Q [B, V, d] f32 query views, cells [B * V, ma] their probed cells
 * (gift_quantize; < 0 or >= K: none), the F-IF's cell_off [K+1], post_ord [P]
 * (global ordinals), f32 features [P, d]; out [B, n_local] f64 = per shape
 * the mean over the V views of the best f64 similarity in the probed cells
 * (all-zero views contribute 0).  ws: gift_fif_score_f64_ws_bytes(B, V,
 * n_local) bytes (per-(view, shape) maxima). */
size_t gift_fif_score_f64_ws_bytes(int32_t B, int32_t V, int64_t n_local);
int gift_fif_score_f64(const float* Q, int32_t B, int32_t V, int32_t d, const int32_t* cells,
                       int32_t ma, int32_t K, const int64_t* cell_off, const int32_t* post_ord,
                       const float* feat, int64_t ord_base, int64_t n_local, int32_t mode,
                       double sigma, void* ws, size_t ws_bytes, double* out, void* stream);

/* ---- evaluation ranks: the 1-based positions evaluate_index /
 * exact_baseline_report give each relevant shape (index.py:317-357): for
 * each query row b of scores [B, N] and each rel[b, r] >= 0,
 * out_rank[b, r] = 1 + #{i != self_local[b] : key_i before key_j}, key =
 * (score desc, idrank asc); NaN scores are excluded; -1 where rel is -1.
 * R <= 4096. */
int gift_eval_ranks(const double* scores, int32_t B, int64_t N, const int32_t* idrank,
                    const int32_t* self_local, const int32_t* rel, int32_t R,
                    int32_t* out_rank, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GIFT_H_ */
