"""Config-scale restatement of the reference path — TEST INFRASTRUCTURE ONLY.

The same algorithm as `reference_port.py` (and the reference package,
`/root/reference/pkg/src/shapesearch`), reorganised so that it finishes at
BASELINE.json's config sizes on the host cores: every query view's cell
probes are grouped by cell and scored with one f64 GEMM per cell (numpy/BLAS),
instead of one GEMV per (view, cell) as `matching.query_fif` does.  The
arithmetic is the reference's (f64 products of f32 features, clip / max /
sum); only BLAS's summation order differs (~1e-16 relative).  Pinned to the
loop restatement and the reference goldens by tests/test_oracle_golden.py.

Used by tests/ (config-scale parity) and by bench.py's `--impl reference`
index build.  Never imported by the product package.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .reference_port import (Act, Sif, aggregate, make_activation, mean_activation,
                             sqdist_exact)

__all__ = ["quantize_many_mt", "fif_lists", "fif_scores_many", "topk_stable",
           "activations_from_scores", "build_context", "rerank_query", "rank_final",
           "OracleCsrIndex"]


def _threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


# ----------------------------------------------------------------- quantize
def quantize_many_mt(centroids, X, ma: int = 1, chunk: int = 8192, threads: int | None = None):
    """codebook.py:111-124 for many rows, bit-identical to the per-row
    reference (the f64 GEMM shortlist + exact numpy-order recheck of
    `reference_port.quantize_many`), chunks spread over host threads (the
    GEMM and the C recheck release the GIL)."""
    from .reference_port import quantize_many

    X = np.asarray(X)
    n = X.shape[0]
    if n == 0:
        return np.zeros((0, ma), dtype=np.int64)
    threads = threads or _threads()
    parts = [(s, min(n, s + chunk)) for s in range(0, n, chunk)]
    out = np.empty((n, ma), dtype=np.int64)

    def run(p):
        s, e = p
        out[s:e] = quantize_many(centroids, np.asarray(X[s:e], dtype=np.float64), ma)

    if len(parts) == 1 or threads == 1:
        for p in parts:
            run(p)
    else:
        from threadpoolctl import threadpool_limits

        with threadpool_limits(1), ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, parts))
    return out


# ----------------------------------------------------------------- F-IF
def fif_lists(views, assign, K: int):
    """matching.py:106-133 as CSR: every non-zero view of shape o (in shape-
    major, view-minor order) appended to the list of its cell.  views:
    [N, V, d] (f32 or f16), assign: [N, V] cell per view (ignored for zero
    views).  Returns (cell_off [K+1] i64, post_ord [P] i32, rows [P] i64 =
    flat view index o*V + v) -- features are views.reshape(-1, d)[rows]."""
    N, V = assign.shape
    nz = np.asarray(views).reshape(N * V, -1).any(axis=1)
    flat = np.flatnonzero(nz)
    cells = np.asarray(assign).reshape(-1)[flat]
    order = np.argsort(cells, kind="stable")  # stable: (ordinal, view) order kept per cell
    rows = flat[order]
    cell_off = np.zeros(K + 1, dtype=np.int64)
    np.add.at(cell_off, cells + 1, 1)
    cell_off = np.cumsum(cell_off)
    return cell_off, (rows // V).astype(np.int32), rows.astype(np.int64)


def fif_scores_many(cell_off, post_ord, feat_rows, Q, q_cells, n_shapes: int,
                    similarity: str = "cosine", sigma: float = 0.5, vq=None,
                    threads: int | None = None, pnorm2=None, cell_chunk: int = 1 << 17,
                    shape_base: int = 0, return_best: bool = False) -> np.ndarray:
    """matching.py:136-161 for a batch of queries.

    cell_off/post_ord: the F-IF lists (ordinals ascending inside a cell, as
    build_fif appends them); feat_rows(p0, p1) -> [p1 - p0, d] features of
    posting rows p0..p1 (any float dtype, widened to f64 like `F_e @ row`);
    Q: [B, V, d] query views; q_cells: [B, V, ma] the views' cells (quantize;
    rows of zero views are skipped, matching.py:150-151); vq: views per query
    to divide by (default V: `total / q.shape[0]`).  similarity "cosine" =
    clip(q.p, 0, 1) (matching.py:158); "gaussian" = exp(-|q - p|^2 / sigma^2)
    via |q|^2 + |p|^2 - 2 q.p in f64 (north_star kernel, D1); pnorm2:
    optional [P] f64 |p|^2 per posting row.  Cells are scored in chunks of
    cell_chunk postings (a shape split across chunks keeps its max).  The
    shapes are ordinals shape_base .. shape_base + n_shapes (a block of the
    database).  Returns f64 [B, n_shapes] (never-visited shapes score
    exactly 0), or with return_best the per-view maxima [B, V, n_shapes]."""
    Q = np.asarray(Q)
    B, V, d = Q.shape
    ma = q_cells.shape[2]
    Qf = Q.reshape(B * V, d).astype(np.float64)
    live = Qf.any(axis=1)
    best = np.zeros((B * V, n_shapes), dtype=np.float64)
    rows = np.repeat(np.arange(B * V), ma)
    cells = np.asarray(q_cells).reshape(-1).astype(np.int64)
    keep = live[rows] & (cells >= 0)
    rows, cells = rows[keep], cells[keep]
    order = np.argsort(cells, kind="stable")
    rows, cells = rows[order], cells[order]
    bounds = np.flatnonzero(np.r_[True, cells[1:] != cells[:-1], True]) if len(cells) else [0]
    inv_s2 = 1.0 / (sigma * sigma)
    qn2 = (Qf * Qf).sum(axis=1)
    work = []
    for i in range(len(bounds) - 1):
        c = int(cells[bounds[i]])
        p0, p1 = int(cell_off[c]), int(cell_off[c + 1])
        for a0 in range(p0, p1, cell_chunk):
            work.append((i, a0, min(p1, a0 + cell_chunk)))

    def chunk_best(item):
        i, p0, p1 = item
        F = np.asarray(feat_rows(p0, p1), dtype=np.float64)
        r = rows[bounds[i]:bounds[i + 1]]
        G = Qf[r] @ F.T
        if similarity == "cosine":
            S = np.clip(G, 0.0, 1.0)
        elif similarity == "gaussian":
            pn = (F * F).sum(axis=1) if pnorm2 is None else pnorm2[p0:p1]
            S = np.exp(-np.maximum(qn2[r][:, None] + pn[None, :] - 2.0 * G, 0.0) * inv_s2)
        else:
            raise ValueError(f"unknown similarity {similarity!r}")
        o = np.asarray(post_ord[p0:p1])
        starts = np.flatnonzero(np.r_[True, o[1:] != o[:-1]])
        return r, o[starts] - shape_base, np.maximum.reduceat(S, starts, axis=1)

    def merge(res):
        r, shapes, M = res
        ix = np.ix_(r, shapes)
        best[ix] = np.maximum(best[ix], M)

    threads = threads or _threads()
    if threads == 1 or len(work) < 4:
        for item in work:
            merge(chunk_best(item))
    else:
        from threadpoolctl import threadpool_limits

        # one BLAS thread per chunk GEMM, chunks spread over the host threads
        with threadpool_limits(1), ThreadPoolExecutor(threads) as ex:
            for res in ex.map(chunk_best, work):
                merge(res)
    if return_best:
        return best.reshape(B, V, n_shapes)
    total = best.reshape(B, V, n_shapes).sum(axis=1)
    div = np.full(B, float(V)) if vq is None else np.asarray(vq, dtype=np.float64)
    return total / div[:, None]


# ----------------------------------------------------------------- selection
def topk_stable(S: np.ndarray, k: int):
    """Per row the k best entries by (score desc, ordinal asc) --
    np.lexsort((arange(n), -s))[:k] of rerank.py:74 / :86, vectorised:
    argpartition, then the boundary ties resolved by ordinal."""
    S = np.asarray(S, dtype=np.float64)
    n, N = S.shape
    k = min(k, N)
    if k == 0:
        return np.zeros((n, 0), dtype=np.int64)
    neg = -S
    part = np.argpartition(neg, k - 1, axis=1)[:, :k]
    kth = np.take_along_axis(neg, part, axis=1).max(axis=1)
    out = np.empty((n, k), dtype=np.int64)
    for r in range(n):
        row = neg[r]
        better = np.flatnonzero(row < kth[r])
        ties = np.flatnonzero(row == kth[r])[: k - len(better)]
        sel = np.concatenate([better, ties])
        out[r] = sel[np.lexsort((sel, row[sel]))]
    return out


def activations_from_scores(S: np.ndarray, k1: int, k2: int):
    """build_activation (rerank.py:64-75) and top_neighbors (:78-87) of each
    score row: (list[Act], list[list[int]])."""
    kk = max(k1, k2)
    top = topk_stable(S, kk)
    acts, nbrs = [], []
    for r in range(S.shape[0]):
        t = top[r]
        v = S[r, t]
        acts.append(make_activation(t[:k1], v[:k1]))
        nbrs.append([int(i) for i, x in zip(t[:k2], v[:k2]) if x > 0.0])
    return acts, nbrs


def build_context(raw, nbrs, alpha: float = 0.5):
    """index.py:211-218 with one channel duplicated (D4): co_augment of the
    raw activations over the neighbourhoods (rerank.py:114-125), aggregate of
    identical channels (identity, rerank.py:142-146), build_sif
    (rerank.py:187-208).  Returns (final activations, Sif)."""
    final = [mean_activation(raw, nb) for nb in nbrs]
    final = [aggregate(f, f, alpha) for f in final]
    n = len(final)
    cnt = np.zeros(n + 1, dtype=np.int64)
    for a in final:
        np.add.at(cnt, a.idx + 1, 1)
    off = np.cumsum(cnt)
    ords = np.empty(off[-1], dtype=np.int32)
    vals = np.empty(off[-1], dtype=np.float64)
    fill = off[:-1].copy()
    for j, a in enumerate(final):  # owners ascending inside every entry
        pos = fill[a.idx]
        ords[pos] = j
        vals[pos] = a.val
        fill[a.idx] += 1
    sif = Sif(norms=np.array([a.norm for a in final], dtype=np.float64),
              entry_ordinals=[ords[off[i]:off[i + 1]] for i in range(n)],
              entry_values=[vals[off[i]:off[i + 1]] for i in range(n)])
    return final, sif


def build_context_arrays(raw_idx, raw_val, raw_cnt, nbr, alpha: float = 0.5):
    """`build_context` without Python loops, for config-scale N: the same
    arithmetic in the same order.  raw_* : [N, k1] activation rows (indices
    ascending, -1 / 0 padded, cnt valid entries); nbr: [N, k2] neighbour
    lists (best first, -1 padded).

    mean_activation (rerank.py:90-100): each coordinate's values are summed
    in neighbour order starting from 0.0 (dict `acc.get(i, 0.0) + v`), then
    divided by the neighbour count; make_activation sorts by coordinate and
    keeps values > 0 with the sequential norm (rerank.py:24-61); aggregate of
    identical channels is the identity (v1 == v2, rerank.py:142-146); the
    S-IF lists owners ascending per coordinate (rerank.py:187-208).
    Returns (final_idx, final_val, final_cnt, norms, Sif)."""
    raw_idx = np.asarray(raw_idx)
    raw_val = np.asarray(raw_val, dtype=np.float64)
    nbr = np.asarray(nbr)
    N, k1 = raw_idx.shape
    k2 = nbr.shape[1]
    # (owner j, neighbour slot t, entry e) flattened in neighbour order
    j = np.repeat(np.arange(N), k2 * k1)
    t = np.tile(np.repeat(np.arange(k2), k1), N)
    q = nbr[j, t]
    e = np.tile(np.arange(k1), N * k2)
    ok = q >= 0
    qq = np.where(ok, q, 0)
    ok &= e < np.asarray(raw_cnt)[qq]
    j, t, qq, e = j[ok], t[ok], qq[ok], e[ok]
    coord = raw_idx[qq, e].astype(np.int64)
    val = raw_val[qq, e]
    order = np.lexsort((t, coord, j))  # by owner, coordinate, then neighbour order
    j, coord, val = j[order], coord[order], val[order]
    first = np.r_[True, (j[1:] != j[:-1]) | (coord[1:] != coord[:-1])]
    gid = np.cumsum(first) - 1
    ng = int(gid[-1]) + 1 if len(gid) else 0
    pos_in = np.arange(len(gid)) - np.flatnonzero(first)[gid]
    acc = np.zeros(ng)
    for r in range(int(pos_in.max()) + 1 if len(pos_in) else 0):  # sequential per coordinate
        m = pos_in == r
        acc[gid[m]] = acc[gid[m]] + val[m]
    g_owner = j[first]
    g_coord = coord[first]
    cnt_nb = (nbr >= 0).sum(axis=1).astype(np.float64)
    g_val = acc / cnt_nb[g_owner]
    keep = g_val > 0.0
    g_owner, g_coord, g_val = g_owner[keep], g_coord[keep], g_val[keep]
    fcnt = np.bincount(g_owner, minlength=N)
    fstart = np.r_[0, np.cumsum(fcnt)]
    cap = max(1, int(fcnt.max()) if N else 1)
    pos = np.arange(len(g_owner)) - fstart[g_owner]
    fidx = np.full((N, cap), -1, dtype=np.int64)
    fval = np.zeros((N, cap))
    fidx[g_owner, pos] = g_coord
    fval[g_owner, pos] = g_val
    norms = np.zeros(N)
    for r in range(cap):  # _seq_sum: left to right from 0.0
        norms = norms + fval[:, r]
    # S-IF: owners ascending within each coordinate
    o2 = np.lexsort((g_owner, g_coord))
    sc, so, sv = g_coord[o2], g_owner[o2], g_val[o2]
    off = np.r_[0, np.cumsum(np.bincount(sc, minlength=N))]
    sif = Sif(norms=norms,
              entry_ordinals=[so[off[i]:off[i + 1]].astype(np.int32) for i in range(N)],
              entry_values=[sv[off[i]:off[i + 1]] for i in range(N)])
    return fidx, fval, fcnt, norms, sif


def rerank_query(raw, sif: Sif, scores: np.ndarray, k2: int, alpha: float = 0.5):
    """index.py:249-258 (duplicated channel): neighbours from the query's own
    scores, mean of their raw activations, aggregate, query_sif."""
    from .reference_port import query_sif, top_neighbors

    nb = top_neighbors(scores, k2)
    f = mean_activation(raw, nb)
    return query_sif(sif, aggregate(f, f, alpha))


def rank_final(final_scores: np.ndarray, ids, self_id: str, top_k: int):
    """index.py:288-294: lexsort((ids, not_self, -final))[:top_k]."""
    from .reference_port import lexsort_rank

    return lexsort_rank(final_scores, ids, self_id, top_k)


class OracleCsrIndex:
    """A single-channel (duplicated, D4) oracle index over CSR F-IF lists,
    built on the host at config scale: `from_views` quantizes every view
    (bit-exact), lays out the lists and runs the DB self-join (every shape's
    stored views as a query, index.py:196-210) in blocks of shapes."""

    def __init__(self, centroids, cell_off, post_ord, feat_rows, ma, k1, k2, similarity,
                 sigma, n_shapes, alpha=0.5):
        self.C = np.asarray(centroids, dtype=np.float32)
        self.cell_off, self.post_ord, self.feat = cell_off, post_ord, feat_rows
        self.ma, self.k1, self.k2 = ma, k1, k2
        self.similarity, self.sigma, self.alpha = similarity, sigma, alpha
        self.n = n_shapes
        self.feat64 = np.asarray(feat_rows, dtype=np.float64)  # F_e widened once
        self.pnorm2 = (self.feat64 * self.feat64).sum(axis=1)

    def feat_rows(self, p0, p1):
        return self.feat64[p0:p1]

    @classmethod
    def from_views(cls, views, centroids, ma, k1, k2, similarity="cosine", sigma=0.5,
                   assign=None, block=128, self_join=True):
        """assign: optional [N, V, >= 1] nearest cells of every view (best
        first); computed bit-exactly here otherwise (with max(ma, 1) columns,
        reused by the self-join's multiple assignment)."""
        views = np.asarray(views)
        N, V, d = views.shape
        C = np.asarray(centroids, dtype=np.float32)
        if assign is None:
            assign = quantize_many_mt(C, views.reshape(N * V, d), ma).reshape(N, V, ma)
        assign = np.asarray(assign).reshape(N, V, -1)
        cell_off, post_ord, rows = fif_lists(views, assign[:, :, 0], C.shape[0])
        feat = views.reshape(N * V, d)[rows]
        self = cls(C, cell_off, post_ord, feat, ma, k1, k2, similarity, sigma, N)
        self.assign = assign
        self.rows = rows
        self.views = views
        if self_join:
            self.self_join(block)
        return self

    def scores(self, Q, q_cells=None, vq=None):
        Q = np.asarray(Q)
        if q_cells is None:
            B, V, d = Q.shape
            q_cells = quantize_many_mt(self.C, Q.reshape(B * V, d), self.ma).reshape(B, V, self.ma)
            q_cells = np.where(Q.any(axis=2)[:, :, None], q_cells, -1)
        return fif_scores_many(self.cell_off, self.post_ord, self.feat_rows, Q, q_cells, self.n,
                               self.similarity, self.sigma, vq=vq, pnorm2=self.pnorm2)

    def self_join(self, block=128):
        """index.py:196-210: raw activations and neighbour lists of every DB
        shape, queried with its full view matrix (`vs.matrix(ch)`: zero views
        included, so the mean divides by V, index.py:198-201); then
        co-augment and the S-IF."""
        N, V, d = self.views.shape
        cells = self.assign[:, :, :self.ma] if self.assign.shape[2] >= self.ma else None
        raw, nbrs = [], []
        for b0 in range(0, N, block):
            b1 = min(N, b0 + block)
            Q = self.views[b0:b1]
            qc = None if cells is None else np.where(Q.any(axis=2)[:, :, None],
                                                     cells[b0:b1], -1)
            S = self.scores(Q, q_cells=qc)
            a, nb = activations_from_scores(S, self.k1, self.k2)
            raw += a
            nbrs += nb
        self.raw, self.nbrs = raw, nbrs
        self.final, self.sif = build_context(raw, nbrs, self.alpha)
        return self
