"""numpy restatement of the reference GIFT query path — TEST INFRASTRUCTURE ONLY.

Follows `/root/reference/pkg/src/shapesearch` (cited as file:line).  See
oracle/__init__.py for the import rules and the pinning status.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "quantize", "quantize_many", "Fif", "build_fif", "query_fif", "Act",
    "seq_sum", "make_activation", "build_activation", "top_neighbors",
    "mean_activation", "co_augment", "aggregate", "Sif", "build_sif",
    "query_sif", "jaccard_dense", "OracleIndex", "lexsort_rank",
    "oracle_lib", "train_codebook",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libgiftoracle.so")
_lib = None


def build_oracle_lib(force: bool = False) -> str:
    """Compile oracle/pairwise.c (no FMA contraction) into oracle/_build."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    src = os.path.join(_HERE, "pairwise.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-o", _LIB_PATH, src])
    return _LIB_PATH


def oracle_lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_oracle_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.gift_oracle_sqdist.restype = None
        lib.gift_oracle_sqdist.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                           ctypes.c_int64, ctypes.c_void_p]
        _lib = lib
    return _lib


# --------------------------------------------------------------- quantize
def quantize(centroids, x, ma: int = 1) -> np.ndarray:
    """codebook.py:111-124 — ma nearest centroids by f64 direct-difference
    squared distance (numpy pairwise sum), stable argsort (ties -> lower)."""
    c64 = np.asarray(centroids, dtype=np.float32).astype(np.float64)
    x64 = np.asarray(x, dtype=np.float64).ravel()
    if x64.shape[0] != c64.shape[1]:
        raise ValueError(f"vector dim {x64.shape[0]} != codebook dim {c64.shape[1]}")
    if not 1 <= ma <= c64.shape[0]:
        raise ValueError(f"ma must be in [1, {c64.shape[0]}]")
    diffs = c64 - x64
    d2 = (diffs * diffs).sum(axis=1)
    return np.argsort(d2, kind="stable")[:ma]


def sqdist_exact(centroids, X, cand=None) -> np.ndarray:
    """Bit-exact (numpy-order) d2 via the C helper; cand: (n, m) candidate ids."""
    C = np.ascontiguousarray(centroids, dtype=np.float32)
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    K = C.shape[0]
    lib = oracle_lib()
    if cand is None:
        out = np.empty((n, K), dtype=np.float64)
        lib.gift_oracle_sqdist(X.ctypes.data, n, d, C.ctypes.data, K, None, K, out.ctypes.data)
    else:
        cand = np.ascontiguousarray(cand, dtype=np.int64)
        m = cand.shape[1]
        out = np.empty((n, m), dtype=np.float64)
        lib.gift_oracle_sqdist(X.ctypes.data, n, d, C.ctypes.data, K, cand.ctypes.data, m,
                               out.ctypes.data)
    return out


def quantize_many(centroids, X, ma: int = 1, chunk: int = 4096) -> np.ndarray:
    """Row-wise `quantize` for many vectors, bit-identical to the per-row
    reference: an f64 GEMM shortlist (error << margin) followed by the exact
    numpy-order distance of every shortlisted centroid (C helper)."""
    C = np.asarray(centroids, dtype=np.float32)
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    K = C.shape[0]
    if not 1 <= ma <= K:
        raise ValueError(f"ma must be in [1, {K}]")
    out = np.empty((n, ma), dtype=np.int64)
    c64 = C.astype(np.float64)
    cn2 = (c64 * c64).sum(axis=1)
    cmax = float(np.sqrt(cn2.max())) if K else 0.0
    m = min(K, ma + 8)
    for s in range(0, n, chunk):
        Xc = X[s:s + chunk]
        xn2 = (Xc * Xc).sum(axis=1)
        approx = cn2[None, :] - 2.0 * (Xc @ c64.T) + xn2[:, None]
        scale = (np.sqrt(xn2) + cmax) ** 2
        margin = 1e-9 * scale + 1e-300
        if m < K:
            part = np.argpartition(approx, m - 1, axis=1)[:, :m]
        else:
            part = np.tile(np.arange(K), (len(Xc), 1))
        pa = np.take_along_axis(approx, part, axis=1)
        order = np.argsort(pa, axis=1, kind="stable")
        part = np.take_along_axis(part, order, axis=1)
        pa = np.take_along_axis(pa, order, axis=1)
        kth = pa[:, ma - 1]
        # every centroid within 2*margin of the ma-th must be in the shortlist
        outside_min = np.full(len(Xc), np.inf)
        if m < K:
            mask = np.ones_like(approx, dtype=bool)
            np.put_along_axis(mask, part, False, axis=1)
            outside_min = np.where(mask, approx, np.inf).min(axis=1)
        safe = outside_min > kth + 2 * margin
        exact = sqdist_exact(C, Xc, part)
        for i in range(len(Xc)):
            if safe[i]:
                cand, dd = part[i], exact[i]
            else:
                cand = np.arange(K)
                dd = sqdist_exact(C, Xc[i:i + 1])[0]
            o = np.lexsort((cand, dd))
            out[s + i] = cand[o[:ma]]
    return out


# --------------------------------------------------------------- F-IF
@dataclass
class Fif:
    """matching.py:64-103 — K lists of (ordinal int32, feature f32[d])."""
    centroids: np.ndarray
    n_shapes: int
    entry_ordinals: list = field(default_factory=list)
    entry_features: list = field(default_factory=list)

    @property
    def total_postings(self) -> int:
        return int(sum(len(o) for o in self.entry_ordinals))

    def pnorm2(self, e: int) -> np.ndarray:
        cache = self.__dict__.setdefault("_pn", {})
        if e not in cache:
            F = self.entry_features[e].astype(np.float64)
            cache[e] = (F * F).sum(axis=1)
        return cache[e]

    def shape_matrix(self, ordinal: int) -> np.ndarray:
        """matching.py:94-103 — cell-major gather of one shape's views."""
        rows = [f[o == ordinal] for o, f in zip(self.entry_ordinals, self.entry_features)
                if (o == ordinal).any()]
        return np.concatenate(rows, axis=0)


def build_fif(mats, centroids, assign=None) -> Fif:
    """matching.py:106-133 — each non-zero view appended, in shape-major /
    view-minor order, to the list of its nearest centroid (ma = 1).
    `assign` may carry precomputed nearest cells (one per view)."""
    C = np.asarray(centroids, dtype=np.float32)
    K, d = C.shape
    ords, rows, cells = [], [], []
    flat = []
    for o, mat in enumerate(mats):
        mat = np.asarray(mat, dtype=np.float32)
        if mat.shape[1] != d:
            raise ValueError("dimension mismatch")
        for r, row in enumerate(mat):
            if not row.any():
                continue
            flat.append((o, r))
            ords.append(o)
            rows.append(row)
    if assign is None:
        cells = [int(quantize(C, row, 1)[0]) for row in rows]
    else:
        cells = [int(assign[o][r]) for (o, r) in flat]
    fif = Fif(centroids=C, n_shapes=len(mats))
    buckets_o = [[] for _ in range(K)]
    buckets_f = [[] for _ in range(K)]
    for o, row, c in zip(ords, rows, cells):
        buckets_o[c].append(o)
        buckets_f[c].append(row)
    for bo, bf in zip(buckets_o, buckets_f):
        fif.entry_ordinals.append(np.asarray(bo, dtype=np.int32))
        fif.entry_features.append(np.stack(bf).astype(np.float32) if bf
                                  else np.zeros((0, d), dtype=np.float32))
    return fif


def query_fif(fif: Fif, query_views, ma: int = 2, similarity: str = "cosine",
              sigma: float = 0.5, cells=None) -> np.ndarray:
    """matching.py:136-161 — mean over query views of the best similarity
    among the postings of the view's ma nearest cells; unvisited shapes 0.

    similarity="gaussian" substitutes s = exp(-|q-p|^2 / sigma^2) (f64 direct
    difference) for clip(q.p, 0, 1) at matching.py:158 — the north-star kernel
    (SURVEY.md D1); everything else is unchanged.  `cells` may carry the
    precomputed (Vq, ma) quantize result."""
    q = np.asarray(query_views, dtype=np.float64)
    if q.ndim != 2 or q.shape[0] == 0:
        raise ValueError("view set is empty")
    n = fif.n_shapes
    total = np.zeros(n, dtype=np.float64)
    inv_s2 = 1.0 / (sigma * sigma)
    for vi, row in enumerate(q):
        if not row.any():
            continue
        entries = quantize(fif.centroids, row, ma) if cells is None else cells[vi]
        best = np.zeros(n, dtype=np.float64)
        for e in entries:
            ords = fif.entry_ordinals[int(e)]
            if len(ords) == 0:
                continue
            F = fif.entry_features[int(e)]
            if similarity == "cosine":
                sims = np.clip(F @ row, 0.0, 1.0)
            elif similarity == "gaussian_expanded":
                # same kernel via |q|^2 + |p|^2 - 2 q.p (one GEMV per cell, the
                # reference's cost profile); used only for CPU-baseline timing
                pn = fif.pnorm2(int(e))
                d2 = np.maximum(row @ row + pn - 2.0 * (F @ row), 0.0)
                sims = np.exp(-d2 * inv_s2)
            else:
                diff = F.astype(np.float64) - row
                sims = np.exp(-(diff * diff).sum(axis=1) * inv_s2)
            np.maximum.at(best, ords, sims)
        total += best
    return total / q.shape[0]


# --------------------------------------------------------------- activations
@dataclass
class Act:
    """rerank.py:34-48 — sparse vector over shape ordinals."""
    idx: np.ndarray   # int64 strictly ascending
    val: np.ndarray   # f64 > 0
    norm: float

    def as_dict(self):
        return dict(zip(self.idx.tolist(), self.val.tolist()))


def seq_sum(values) -> float:
    """rerank.py:24-31 — left-to-right f64 sum from 0.0."""
    t = 0.0
    for v in values:
        t += float(v)
    return t


def make_activation(indices, values) -> Act:
    """rerank.py:51-61."""
    i = np.asarray(indices, dtype=np.int64)
    v = np.asarray(values, dtype=np.float64)
    o = np.argsort(i, kind="stable")
    i, v = i[o], v[o]
    keep = v > 0.0
    i, v = i[keep], v[keep]
    return Act(i, v, seq_sum(v))


def _rank_desc(scores) -> np.ndarray:
    # np.lexsort((arange(n), -scores)) == stable argsort of -scores
    return np.argsort(-np.asarray(scores, dtype=np.float64), kind="stable")


def build_activation(scores, k1: int) -> Act:
    """rerank.py:64-75 — top-k1 by (score desc, ordinal asc), positives only."""
    s = np.asarray(scores, dtype=np.float64)
    if k1 < 1:
        raise ValueError("k1 must be >= 1")
    top = _rank_desc(s)[: min(k1, len(s))]
    return make_activation(top, s[top])


def top_neighbors(scores, k2: int) -> list:
    """rerank.py:78-87 — best-first ordinals of the top-k2 positive scores."""
    s = np.asarray(scores, dtype=np.float64)
    top = _rank_desc(s)[: min(k2, len(s))]
    return [int(i) for i in top if s[i] > 0.0]


def mean_activation(acts, neighbor_list) -> Act:
    """rerank.py:90-100 — dict accumulation in neighbour order."""
    if not neighbor_list:
        return make_activation([], [])
    acc: dict = {}
    for q in neighbor_list:
        a = acts[q]
        for i, v in zip(a.idx.tolist(), a.val.tolist()):
            acc[i] = acc.get(i, 0.0) + v
    cnt = float(len(neighbor_list))
    keys = sorted(acc)
    return make_activation(keys, [acc[k] / cnt for k in keys])


def co_augment(acts1, acts2, nbr1, nbr2):
    """rerank.py:114-125 — channel 1 over channel-2 neighbourhoods and vice
    versa, reading pre-update activations."""
    out1 = [mean_activation(acts1, nbr2[q]) for q in range(len(acts1))]
    out2 = [mean_activation(acts2, nbr1[q]) for q in range(len(acts2))]
    return out1, out2


def aggregate(f1: Act, f2: Act, alpha: float = 0.5) -> Act:
    """rerank.py:128-147 — generalized mean over the union support."""
    if alpha <= 0.0:
        raise ValueError("alpha must be > 0")
    u = np.union1d(f1.idx, f2.idx)
    v1 = np.zeros(len(u))
    v2 = np.zeros(len(u))
    v1[np.searchsorted(u, f1.idx)] = f1.val
    v2[np.searchsorted(u, f2.idx)] = f2.val
    mixed = ((np.power(v1, alpha) + np.power(v2, alpha)) / 2.0) ** (1.0 / alpha)
    return make_activation(u, np.where(v1 == v2, v1, mixed))


def jaccard_dense(fq: Act, fp: Act) -> float:
    """rerank.py:150-162."""
    if len(fq.idx) == 0 and len(fp.idx) == 0:
        return 0.0
    _, qi, pi = np.intersect1d(fq.idx, fp.idx, return_indices=True)
    smin = seq_sum(np.minimum(fq.val[qi], fp.val[pi]))
    smax = fq.norm + fp.norm - smin
    return 0.0 if smax <= 0.0 else smin / smax


@dataclass
class Sif:
    """rerank.py:165-184."""
    norms: np.ndarray
    entry_ordinals: list
    entry_values: list

    @property
    def n_shapes(self) -> int:
        return len(self.norms)


def build_sif(acts) -> Sif:
    """rerank.py:187-208 — transpose; each entry lists owners ascending."""
    n = len(acts)
    bo = [[] for _ in range(n)]
    bv = [[] for _ in range(n)]
    for j, a in enumerate(acts):
        for i, v in zip(a.idx.tolist(), a.val.tolist()):
            if not 0 <= i < n:
                raise ValueError(f"activation coordinate {i} outside database of {n}")
            bo[i].append(j)
            bv[i].append(v)
    return Sif(norms=np.array([a.norm for a in acts], dtype=np.float64),
               entry_ordinals=[np.asarray(o, dtype=np.int32) for o in bo],
               entry_values=[np.asarray(v, dtype=np.float64) for v in bv])


def query_sif(sif: Sif, fq: Act) -> np.ndarray:
    """rerank.py:211-230 — acc over the query support in ascending order."""
    n = sif.n_shapes
    acc = np.zeros(n, dtype=np.float64)
    for i, v in zip(fq.idx.tolist(), fq.val.tolist()):
        if i >= n:
            continue
        o = sif.entry_ordinals[i]
        if len(o) == 0:
            continue
        acc[o] += np.minimum(v, sif.entry_values[i])
    out = np.zeros(n, dtype=np.float64)
    t = acc > 0.0
    out[t] = acc[t] / (fq.norm + sif.norms[t] - acc[t])
    return out


def lexsort_rank(scores, ids, self_id, top_k):
    """index.py:288-294 — (score desc, own entry first, id asc)."""
    ids = np.asarray(ids)
    not_self = ids != self_id
    order = np.lexsort((ids, not_self, -np.asarray(scores, dtype=np.float64)))
    return order[: min(top_k, len(ids))]


# --------------------------------------------------------------- pipeline
class OracleIndex:
    """index.py:146-227 (build) and :230-314 (query) over feature matrices.

    `mats_a` / `mats_b`: per-shape (V, d) view matrices of channels A and B;
    mats_b=None feeds the one feature set as both channels and
    computes the F-IF once (`single_channel=True`) or twice (as the
    reference does).  Codebooks are given (D3: sampled, not trained)."""

    def __init__(self, mats_a, centroids_a, shape_ids, *, mats_b=None, centroids_b=None,
                 ma=2, k1=10, k2=4, alpha=0.5, similarity="cosine", sigma=0.5,
                 single_channel=True, assign_a=None, assign_b=None, build_sif_now=True):
        self.shape_ids = list(shape_ids)
        self.ma, self.k1, self.k2, self.alpha = ma, k1, k2, alpha
        self.similarity, self.sigma = similarity, sigma
        self.dup = mats_b is None
        self.single = single_channel and self.dup
        self.mats = {"A": mats_a, "B": mats_a if self.dup else mats_b}
        cb = {"A": centroids_a, "B": centroids_a if centroids_b is None else centroids_b}
        self.fifs = {"A": build_fif(mats_a, cb["A"], assign_a)}
        if self.single:
            self.fifs["B"] = self.fifs["A"]
        else:
            self.fifs["B"] = build_fif(self.mats["B"], cb["B"],
                                       assign_a if self.dup else assign_b)
        if build_sif_now:
            self.build_context()

    @classmethod
    def from_parts(cls, shape_ids, centroids, entry_ordinals, entry_features, raw, sif, *,
                   ma, k1, k2, alpha=0.5, similarity="cosine", sigma=0.5, single_channel=True):
        """Assemble an oracle index over one feature set (duplicated channel,
        D4) from given lists (oracle.scale's host build, or parity-verified
        GPU-built lists).  single_channel=False scores channel B again, as
        the reference does with two identical channels ("as-is")."""
        self = cls.__new__(cls)
        self.shape_ids = list(shape_ids)
        self.ma, self.k1, self.k2, self.alpha = ma, k1, k2, alpha
        self.similarity, self.sigma = similarity, sigma
        self.dup = True
        self.single = single_channel
        fif = Fif(centroids=np.asarray(centroids, dtype=np.float32), n_shapes=len(shape_ids),
                  entry_ordinals=list(entry_ordinals), entry_features=list(entry_features))
        self.fifs = {"A": fif, "B": fif}
        self.raw = {"A": raw, "B": raw}
        self.sif = sif
        return self

    def channel_scores(self, views, ch):
        return query_fif(self.fifs[ch], views, self.ma, self.similarity, self.sigma)

    def build_context(self):
        """index.py:196-218 — DB self-join, raw activations, co-augment, S-IF."""
        n = len(self.shape_ids)
        scores = {"A": [self.channel_scores(self.mats["A"][i], "A") for i in range(n)]}
        scores["B"] = scores["A"] if self.single else [
            self.channel_scores(self.mats["B"][i], "B") for i in range(n)]
        self.db_scores = scores
        self.raw = {ch: [build_activation(scores[ch][i], self.k1) for i in range(n)]
                    for ch in ("A", "B")}
        self.nbrs = {ch: [top_neighbors(scores[ch][i], self.k2) for i in range(n)]
                     for ch in ("A", "B")}
        aug_a, aug_b = co_augment(self.raw["A"], self.raw["B"], self.nbrs["A"], self.nbrs["B"])
        self.final = [aggregate(a, b, self.alpha) for a, b in zip(aug_a, aug_b)]
        self.sif = build_sif(self.final)

    def rerank_scores(self, ch_scores):
        """index.py:249-258."""
        nb = {ch: top_neighbors(ch_scores[ch], self.k2) for ch in ("A", "B")}
        fa = mean_activation(self.raw["A"], nb["B"])
        fb = mean_activation(self.raw["B"], nb["A"])
        return query_sif(self.sif, aggregate(fa, fb, self.alpha))

    def query(self, views_a, views_b=None, self_id="", top_k=10, rerank=True):
        """index.py:261-299 minus rendering: returns ([(id, score)], final)."""
        s = {"A": self.channel_scores(views_a, "A")}
        if self.single:
            s["B"] = s["A"]
        else:
            s["B"] = self.channel_scores(views_a if views_b is None else views_b, "B")
        final = self.rerank_scores(s) if rerank else np.mean([s["A"], s["B"]], axis=0)
        order = lexsort_rank(final, self.shape_ids, self_id, top_k)
        return [(self.shape_ids[i], float(final[i])) for i in order], final

    def query_by_id(self, shape_id, top_k=10, rerank=True):
        """index.py:302-314 — stored views recovered cell-major."""
        o = self.shape_ids.index(shape_id)
        va = self.fifs["A"].shape_matrix(o)
        vb = None if self.single else self.fifs["B"].shape_matrix(o)
        return self.query(va, vb, self_id=shape_id, top_k=top_k, rerank=rerank)


# ------------------------------------------------------------------ codebook training
def _sq_dists(points, centers):
    """codebook.py:37-45: (|x|^2 - 2 x.c) + |c|^2 (BLAS product), clamped at 0."""
    d2 = ((points * points).sum(axis=1)[:, None] - 2.0 * points @ centers.T
          + (centers * centers).sum(axis=1)[None, :])
    np.maximum(d2, 0.0, out=d2)
    return d2


def train_codebook(features, k: int, seed: int = 0, max_iters: int = 50) -> np.ndarray:
    """codebook.py:48-108 restated: k-means++ seeding (rng.integers for the
    first center, rng.choice(n, p=D^2 / sum) per further center, rng.integers
    when every distance is 0), then Lloyd iterations with the empty-cluster
    repair (the largest cluster donates its farthest member) until the
    relative cost change drops under 1e-4.  Returns f32 centroids (k, d)."""
    points = np.asarray(features, dtype=np.float64)
    n = points.shape[0]
    if n < k:
        points = np.tile(points, (-(-k // n), 1))
        n = points.shape[0]
    rng = np.random.default_rng(seed)
    centers = np.empty((k, points.shape[1]), dtype=np.float64)
    centers[0] = points[rng.integers(0, n)]
    closest = _sq_dists(points, centers[:1])[:, 0]
    for i in range(1, k):
        total = closest.sum()
        idx = int(rng.integers(0, n)) if total <= 0.0 else int(rng.choice(n, p=closest / total))
        centers[i] = points[idx]
        np.minimum(closest, _sq_dists(points, centers[i:i + 1])[:, 0], out=closest)
    prev = None
    for _ in range(max_iters):
        d2 = _sq_dists(points, centers)
        lab = d2.argmin(axis=1)
        cost = float(d2[np.arange(n), lab].sum())
        counts = np.bincount(lab, minlength=k)
        for e in np.flatnonzero(counts == 0):
            donor = int(counts.argmax())
            members = np.flatnonzero(lab == donor)
            steal = members[d2[members, donor].argmax()]
            lab[steal] = e
            counts[donor] -= 1
            counts[e] += 1
        new = np.zeros_like(centers)
        np.add.at(new, lab, points)
        centers = new / counts[:, None]
        if prev is not None and abs(prev - cost) / max(prev, 1e-300) < 1e-4:
            break
        prev = cost
    return centers.astype(np.float32)
