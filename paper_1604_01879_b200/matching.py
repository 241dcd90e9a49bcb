"""First inverted file: GPU build and batched scoring.

Mirrors `shapesearch.matching` (matching.py:22-211): the exact set matching
functions (exact_hausdorff_distance, exact_similarity, on libgift's f64
gift_exact_sets), FirstInvertedFile, build_fif, query_fif, save_fif/load_fif.
"""

from __future__ import annotations

import struct
import threading

import numpy as np
import torch

from . import _native as nat
from . import engine as eg
from .codebook import Codebook
from .errors import DimensionMismatch, EmptySet, FormatError

DEFAULT_MA = 2
_TLS = threading.local()


def runner() -> eg.ScoreRunner:
    """The calling thread's scan launcher (its grow-only workspaces are per
    stream; one per thread keeps concurrent callers independent)."""
    r = getattr(_TLS, "runner", None)
    if r is None:
        r = _TLS.runner = eg.ScoreRunner()
    return r


def release_workspaces() -> None:
    """Drop the calling thread's scan launcher and its grow-only workspaces
    (up to the compact buffer's pre-sized worst case per stream): call it
    between large indexes so their HBM goes back to the allocator."""
    _TLS.runner = None


def sim_mode(similarity: str) -> int:
    if similarity == "cosine":
        return nat.SIM_COSINE
    if similarity == "gaussian":
        return nat.SIM_GAUSSIAN
    raise ValueError(f"unknown similarity {similarity!r}")


class FirstInvertedFile:
    """Codeword-indexed postings of (shape ordinal, stored view feature),
    resident on the GPU as a cell-major CSR (engine.DeviceFif).  The
    reference's list attributes are materialized on demand."""

    def __init__(self, codebook: Codebook, shape_ids, n_views: int, dev: eg.DeviceFif):
        self.codebook = codebook
        self.shape_ids = list(shape_ids)
        self.n_views = n_views
        self.dev = dev
        self._host = None

    @property
    def k(self) -> int:
        return self.codebook.k

    @property
    def dim(self) -> int:
        return self.codebook.dim

    @property
    def n_shapes(self) -> int:
        return len(self.shape_ids)

    @property
    def total_postings(self) -> int:
        return self.dev.P

    def _lists(self):
        if self._host is None:
            self._host = self.dev.host_lists()
        return self._host

    @property
    def entry_ordinals(self):
        return self._lists()[0]

    @property
    def entry_features(self):
        return self._lists()[1]

    def shape_matrix(self, ordinal: int) -> np.ndarray:
        """Stored views of one shape, gathered cell-major (matching.py:94-103)."""
        loc = ordinal - self.dev.ord_base
        if not 0 <= loc < self.dev.n_local:
            raise EmptySet(f"shape ordinal {ordinal} has no stored views")
        lo, hi = (int(v) for v in self.dev.shape_off[loc:loc + 2].cpu())
        if hi == lo:
            raise EmptySet(f"shape ordinal {ordinal} has no stored views")
        Q, _vq = self.dev.shape_views(torch.tensor([loc], device=self.dev.device))
        return Q[0].cpu().numpy()


# ------------------------------------------------------------------ exact
def _exact_operand(views):
    """matching.py:22-26 `_as_matrix`: a non-empty 2-D view set (f32 values
    keep f32 storage; anything else is widened to f64 like the reference)."""
    if torch.is_tensor(views):
        views = views.detach().cpu().numpy()
    arr = np.asarray(views)
    if arr.dtype != np.float32:
        arr = arr.astype(np.float64)
    if arr.ndim != 2 or arr.shape[0] == 0:
        raise EmptySet("view set is empty")
    return np.ascontiguousarray(arr)


def exact_set_scores(query_sets, target_sets, q_counts=None, t_counts=None) -> torch.Tensor:
    """Batched exact matching (new): query_sets [B, Vq, d], target_sets [N,
    Vp, d] (host or device, f32/f64; the first q_counts[b] / t_counts[n]
    views of each set are used) -> device f64 [B, N, 3] = (robust Hausdorff,
    standard Hausdorff, exact similarity), matching.py:39-61 for every pair."""
    dev = nat.device()

    def prep(x):
        t = x if torch.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x))
        if t.dtype not in (torch.float32, torch.float64):
            t = t.double()
        return t.to(dev).contiguous()

    Q, P = prep(query_sets), prep(target_sets)
    if Q.dim() != 3 or P.dim() != 3:
        raise ValueError("view sets must be [n_sets, n_views, d]")
    if Q.shape[2] != P.shape[2]:
        raise DimensionMismatch(f"view dims differ: {Q.shape[2]} vs {P.shape[2]}")
    qc = None if q_counts is None else torch.as_tensor(q_counts, dtype=torch.int32).to(dev)
    pc = None if t_counts is None else torch.as_tensor(t_counts, dtype=torch.int32).to(dev)
    B, N = Q.shape[0], P.shape[0]
    out = torch.empty((B, N, 3), dtype=torch.float64, device=dev)
    code = {torch.float32: nat.GIFT_F32, torch.float64: nat.GIFT_F64}
    nat.call("gift_exact_sets", nat.ptr(Q), code[Q.dtype], nat.ptr(qc), B, Q.shape[1],
             nat.ptr(P), code[P.dtype], nat.ptr(pc), N, P.shape[1], Q.shape[2], nat.ptr(out),
             nat.stream_ptr())
    return out


def _exact_pair(query_views, target_views):
    q = _exact_operand(query_views)
    p = _exact_operand(target_views)
    if q.shape[1] != p.shape[1]:
        raise DimensionMismatch(f"view dims differ: {q.shape[1]} vs {p.shape[1]}")
    return exact_set_scores(q[None], p[None])[0, 0].cpu().numpy()


def exact_hausdorff_distance(query_views, target_views, variant: str = "robust") -> float:
    """Exact Hausdorff distance between two view sets with d = 1 - cosine
    (matching.py:39-52): "standard" = max over query views of the min
    distance, "robust" = their mean."""
    if variant not in ("standard", "robust"):
        _exact_pair(query_views, target_views)  # the reference validates the sets first
        raise ValueError(f"unknown variant {variant!r}")
    r = _exact_pair(query_views, target_views)
    return float(r[1] if variant == "standard" else r[0])


def exact_similarity(query_views, target_views) -> float:
    """Mean over query views of the best clamped cosine in the target set
    (matching.py:55-61)."""
    return float(_exact_pair(query_views, target_views)[2])


def _stack_views(viewsets, channel, dim):
    mats = []
    for vs in viewsets:
        mat = vs.matrix(channel)
        if mat.shape[1] != dim:
            raise DimensionMismatch(f"shape {vs.shape_id!r} dim {mat.shape[1]} != codebook dim {dim}")
        mats.append(np.asarray(mat, dtype=np.float32))
    V = max(m.shape[0] for m in mats)
    X = np.zeros((len(mats), V, dim), dtype=np.float32)
    for i, m in enumerate(mats):
        X[i, : m.shape[0]] = m
    return X, V


def build_fif(viewsets, codebook: Codebook, channel: str,
              storage_dtype=torch.float32) -> FirstInvertedFile:
    """Store each non-empty view once, under its nearest codeword
    (matching.py:106-133) — K1 quantize + K2 device radix-sort layout."""
    viewsets = list(viewsets)
    X, V = _stack_views(viewsets, channel, codebook.dim)
    dev = nat.device()
    Xd = torch.from_numpy(X).to(dev).to(storage_dtype)
    d = eg.DeviceFif.build(Xd, codebook.device())
    return FirstInvertedFile(codebook, [vs.shape_id for vs in viewsets], V, d)


def build_fif_from_tensor(X: torch.Tensor, codebook: Codebook, shape_ids,
                          ord_base: int = 0) -> FirstInvertedFile:
    """Build from a device tensor [n, V, d] (f32 or f16 storage)."""
    d = eg.DeviceFif.build(X, codebook.device(), ord_base=ord_base)
    return FirstInvertedFile(codebook, shape_ids, X.shape[1], d)


def _as_query_tensor(query_views, dim):
    if torch.is_tensor(query_views):
        q = query_views
    else:
        arr = np.asarray(query_views, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[0] == 0:
            raise EmptySet("view set is empty")
        q = torch.from_numpy(arr.astype(np.float32))
    if q.dim() != 2 or q.shape[0] == 0:
        raise EmptySet("view set is empty")
    if q.shape[1] != dim:
        raise DimensionMismatch(f"query dim {q.shape[1]} != index dim {dim}")
    return q.to(nat.device(), dtype=torch.float32)


PRECISIONS = ("tc", "f64")
F64_WS_BYTES = 1 << 30  # score_f64: workspace per chunk of queries


def query_fif(fif: FirstInvertedFile, query_views, ma: int = DEFAULT_MA,
              similarity: str = "cosine", sigma: float = 0.5,
              precision: str = "tc") -> np.ndarray:
    """Approximate similarity of one query view set against every shape
    (matching.py:136-161).  Query views are scored as f32 (stored features
    are f32); scores are f64.  precision "tc": the tensor-core scan (1e-5
    relative, the throughput path); "f64": f64 similarities on CUDA cores
    (f64 rounding: the reference's own arithmetic, for small indexes)."""
    q = _as_query_tensor(query_views, fif.dim)
    return query_fif_batch(fif, q[None], ma, similarity, sigma, precision=precision)[0].cpu().numpy()


def query_fif_batch(fif: FirstInvertedFile, Q, ma: int = DEFAULT_MA, similarity: str = "cosine",
                    sigma: float = 0.5, vq=None, precision: str = "tc") -> torch.Tensor:
    """Batched scores: Q [B, V, d] -> device f64 [B, n_local] (new API)."""
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    if not torch.is_tensor(Q):
        Q = torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float32))
    Q = Q.to(nat.device(), dtype=torch.float32)
    if precision == "f64":
        return score_f64(fif.dev, Q, ma, sim_mode(similarity), sigma)
    return runner().score(fif.dev, Q, ma, sim_mode(similarity), sigma, vq=vq)


def score_f64(dev: eg.DeviceFif, Q: torch.Tensor, ma: int, mode: int, sigma: float,
              stream=None) -> torch.Tensor:
    """query_fif's arithmetic in f64 (libgift gift_fif_score_f64): the query
    views' ma cells from the bit-exact quantizer, every probed posting's f64
    similarity, per-(view, shape) max, view-order f64 sums / V."""
    if Q.dim() != 3 or Q.shape[1] == 0:
        raise EmptySet("view set is empty")
    B, V, d = Q.shape
    if d != dev.d:
        raise DimensionMismatch(f"query dim {d} != index dim {dev.d}")
    if not 1 <= ma <= dev.cb.K:
        raise ValueError(f"ma must be in [1, {dev.cb.K}]")
    if dev.feat is None or dev.feat.dtype != torch.float32:
        raise ValueError("the f64 scan needs the index's f32 feature copy")
    Q = Q.contiguous()
    out = torch.empty((B, dev.n_local), dtype=torch.float64, device=Q.device)
    if B == 0 or dev.n_local == 0:
        return out.zero_()
    cells = eg.quantize_rows(dev.cb, Q.view(-1, d), ma, stream=stream)
    # the per-(view, shape) maxima take V n_local 8 bytes per query: queries
    # go in chunks of at most F64_WS_BYTES of them
    lib = nat.lib()
    per_q = max(1, lib.gift_fif_score_f64_ws_bytes(1, V, dev.n_local))
    bc = max(1, min(B, F64_WS_BYTES // per_q))
    ws = torch.empty(-(-lib.gift_fif_score_f64_ws_bytes(bc, V, dev.n_local) // 8),
                     dtype=torch.int64, device=Q.device)
    for b0 in range(0, B, bc):
        nb = min(bc, B - b0)
        wsb = lib.gift_fif_score_f64_ws_bytes(nb, V, dev.n_local)
        nat.call("gift_fif_score_f64", nat.ptr(Q[b0:b0 + nb]), nb, V, d,
                 nat.ptr(cells[b0 * V:(b0 + nb) * V]), ma, dev.cb.K, nat.ptr(dev.cell_off),
                 nat.ptr(dev.post_ord), nat.ptr(dev.feat), dev.ord_base, dev.n_local, mode,
                 float(sigma), nat.ptr(ws), wsb, nat.ptr(out[b0:b0 + nb]), eg._sp(stream))
    return out


def save_fif(fif: FirstInvertedFile, path) -> None:
    """matching.py:164-175 byte layout."""
    ords, feats = fif.entry_ordinals, fif.entry_features
    with open(path, "wb") as fh:
        fh.write(struct.pack("<III", fif.k, fif.dim, fif.n_views))
        fh.write(struct.pack("<I", fif.n_shapes))
        for sid in fif.shape_ids:
            raw = sid.encode("utf-8")
            fh.write(struct.pack("<H", len(raw)))
            fh.write(raw)
        for o, f in zip(ords, feats):
            fh.write(struct.pack("<I", len(o)))
            fh.write(np.asarray(o).astype("<u4").tobytes())
            fh.write(np.asarray(f).astype("<f4").tobytes())


def load_fif(path, codebook: Codebook, storage_dtype=torch.float32) -> FirstInvertedFile:
    """matching.py:178-211: read the lists, rebuild the device layout."""
    data = open(path, "rb").read()
    off = 0

    def take(fmt):
        nonlocal off
        size = struct.calcsize(fmt)
        if off + size > len(data):
            raise FormatError(f"truncated inverted file {path}")
        out = struct.unpack_from(fmt, data, off)
        off += size
        return out

    k, dim, n_views = take("<III")
    if k != codebook.k or dim != codebook.dim:
        raise DimensionMismatch(f"inverted file {path} does not match codebook")
    (n_shapes,) = take("<I")
    ids = []
    for _ in range(n_shapes):
        (n,) = take("<H")
        ids.append(data[off:off + n].decode("utf-8"))
        off += n
    counts, ords, feats = [], [], []
    for _ in range(k):
        (cnt,) = take("<I")
        if off + cnt * 4 * (1 + dim) > len(data):
            raise FormatError(f"truncated inverted file {path}")
        ords.append(np.frombuffer(data, dtype="<u4", count=cnt, offset=off).astype(np.int32))
        off += cnt * 4
        feats.append(np.frombuffer(data, dtype="<f4", count=cnt * dim, offset=off).reshape(cnt, dim))
        off += cnt * dim * 4
        counts.append(cnt)
    dev = nat.device()
    cell_off = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int64, device=dev)
    post_ord = torch.from_numpy(np.concatenate(ords) if ords else np.zeros(0, np.int32)).to(dev)
    feat = torch.from_numpy(np.concatenate(feats) if feats else np.zeros((0, dim), np.float32))
    d = eg.DeviceFif.from_arrays(codebook.device(), cell_off, post_ord,
                                 feat.to(dev).to(storage_dtype), n_shapes, n_views)
    return FirstInvertedFile(codebook, ids, n_views, d)
