"""Pipeline composition on the GPU: index build, batched query, persistence.

Drop-in for `shapesearch.index` (index.py:38-414) on the F-IF + S-IF path:
IndexConfig, IndexBundle, build_index, query, query_by_id, rerank_scores,
save_bundle, load_bundle keep the reference's names, arguments, results and
errors.  New: `build_index_from_views` (explicit feature
tensors and codebooks, D3/D4), `query_batch` / `query_many` (batched and
pipelined queries, D6), and IndexConfig fields `similarity`, `sigma`,
`storage_dtype`, `batch_size` whose defaults reproduce the reference.
"""

from __future__ import annotations

import json
import logging
import os
import threading
import time
from dataclasses import asdict, dataclass, field, fields, replace
from pathlib import Path

import numpy as np
import torch

from . import _native as nat
from . import codebook as cb
from . import engine as eg
from . import features as ft
from . import matching as mt
from . import rerank as rr
from .errors import (AllShapesFailed, ChannelMismatch, EmptyIndex, EmptyManifest, FormatError,
                     Unsupported)

log = logging.getLogger(__name__)

FORMAT_VERSION = "shapesearch-index-1"
CHANNELS = ("A", "B")
CAND_K_MAX = 8  # the reduce's per-range candidates (fif_scan.cu RED_MAXK); larger k2 -> dense path
ACT_MAX_K2 = 64  # act.cu MAX_NBR: neighbours per mean activation
ACT_MAX_E = 1024  # act.cu AM_MAX_E: k1 * k2 staged entries per mean activation
_REFERENCE_FIELDS = ("n_views", "resolution", "grid", "cells", "bins", "codebook_size", "ma",
                     "k1", "k2", "alpha", "seed", "imported")


@dataclass(frozen=True)
class IndexConfig:
    n_views: int = 64
    resolution: int = 64
    grid: int = 8
    cells: int = 4
    bins: int = 8
    codebook_size: int = 256
    ma: int = 2
    k1: int = 10
    k2: int = 4
    alpha: float = 0.5
    seed: int = 0
    imported: bool = False
    # new fields; defaults reproduce the reference
    similarity: str = "cosine"      # or "gaussian" (north-star kernel, D1)
    sigma: float = 0.5
    storage_dtype: str = "float32"  # or "float16" (config 4, D5)
    batch_size: int = 64            # queries per device batch

    def __post_init__(self):
        # index.py:58-64
        if min(self.n_views, self.codebook_size, self.ma, self.k1, self.k2) < 1:
            raise ValueError("all counts must be >= 1")
        if self.alpha <= 0:
            raise ValueError("alpha must be > 0")
        if self.ma > self.codebook_size:
            raise ValueError("ma must not exceed the codebook size")
        if self.similarity not in ("cosine", "gaussian"):
            raise ValueError("similarity must be 'cosine' or 'gaussian'")
        if self.sigma <= 0:
            raise ValueError("sigma must be > 0")
        if self.storage_dtype not in ("float32", "float16"):
            raise ValueError("storage_dtype must be 'float32' or 'float16'")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        # the device mean activation stages k2 lists of <= k1 entries per row
        if self.k2 > ACT_MAX_K2 or self.k1 * self.k2 > ACT_MAX_E:
            raise Unsupported(f"k2 = {self.k2} (max {ACT_MAX_K2}) and k1 * k2 = "
                              f"{self.k1 * self.k2} (max {ACT_MAX_E}) exceed the device "
                              "mean-activation kernel")

    @property
    def torch_storage(self):
        return torch.float16 if self.storage_dtype == "float16" else torch.float32


@dataclass
class IndexBundle:
    config: IndexConfig
    shape_ids: list
    labels: dict
    codebooks: dict
    fifs: dict
    raw_activations: dict
    sif: rr.SecondInvertedFile
    version: str = FORMAT_VERSION
    _engine: object = field(default=None, repr=False, compare=False)

    @property
    def n_shapes(self) -> int:
        return len(self.shape_ids)

    def viewset_matrix(self, channel: str, ordinal: int) -> np.ndarray:
        """Stored view features of one shape (index.py:80-84)."""
        return self.fifs[channel].shape_matrix(ordinal)

    @property
    def engine(self) -> "QueryEngine":
        if self._engine is None:
            self._engine = QueryEngine(self)
        return self._engine


def read_manifest(path) -> list:
    """`path<TAB>label` rows; relative paths resolve against the manifest
    (index.py:87-103)."""
    path = Path(path)
    rows = []
    for line in path.read_text(encoding="utf-8").splitlines():
        line = line.strip()
        if not line:
            continue
        rel, _, label = line.partition("\t")
        rows.append((path.parent / rel, label.strip()))
    if not rows:
        raise EmptyManifest(f"manifest {path} lists no shapes")
    return rows


# ------------------------------------------------------------------ rendering hook
class _Renderer:
    """Mesh rendering + depth descriptors (index.py:106-139) are outside the
    GPU path.  The `shapesearch` shim plugs the reference's own CPU renderer
    in here, so mesh manifests and mesh queries work through this package."""

    compute_viewset = None  # (mesh, config) -> ViewSet
    load_mesh = None        # path -> mesh
    mesh_type = None        # type of mesh query targets


def set_renderer(compute_viewset, load_mesh, mesh_type) -> None:
    _Renderer.compute_viewset = staticmethod(compute_viewset)
    _Renderer.load_mesh = staticmethod(load_mesh)
    _Renderer.mesh_type = mesh_type


def _gather_viewsets(rows, config, jobs: int = 1):
    """index.py:117-139: render every manifest row (in manifest order for any
    job count); rows that fail with a ShapeSearchError / OSError are skipped
    with a warning."""
    from concurrent.futures import ThreadPoolExecutor

    from .errors import ShapeSearchError

    def one(row):
        return _Renderer.compute_viewset(_Renderer.load_mesh(row[0]), config)

    out = []
    if jobs > 1:
        with ThreadPoolExecutor(max_workers=jobs) as pool:
            futs = [pool.submit(one, row) for row in rows]
            for row, fut in zip(rows, futs):
                try:
                    out.append((row, fut.result()))
                except (ShapeSearchError, OSError) as exc:
                    log.warning("skipping shape %s: %s", row[0], exc)
    else:
        for row in rows:
            try:
                out.append((row, one(row)))
            except (ShapeSearchError, OSError) as exc:
                log.warning("skipping shape %s: %s", row[0], exc)
    return out


# ------------------------------------------------------------------ engine
class QueryEngine:
    """Batched device pipeline over one bundle (single GPU or one shard):
    K1 quantize -> K3 F-IF score -> K4 top-k2 -> K5 mean activation
    (-> aggregate) -> K6 S-IF -> K4 final top-k (index.py:230-299)."""

    def __init__(self, bundle: IndexBundle):
        self.b = bundle
        cfg = bundle.config
        self.cfg = cfg
        fa, fb = bundle.fifs.get("A"), bundle.fifs.get("B")
        self.fa = fa.dev if fa is not None else None  # None: list-only index (config 5)
        self.fb = fb.dev if fb is not None else None
        self.dup = fa is fb
        ra, rb = bundle.raw_activations["A"], bundle.raw_activations["B"]
        self.raw_a = rr._rows(ra)
        self.raw_b = self.raw_a if rb is ra else rr._rows(rb)
        self.raw_dup = rb is ra
        self.sif = bundle.sif.dev
        self.n = bundle.n_shapes
        order = sorted(range(self.n), key=lambda i: bundle.shape_ids[i])
        rank = np.empty(self.n, dtype=np.int32)
        rank[np.asarray(order, dtype=np.int64)] = np.arange(self.n, dtype=np.int32)
        self.idrank = torch.from_numpy(rank).to(nat.device())
        self.order = torch.from_numpy(np.asarray(order, dtype=np.int32)).to(nat.device())
        self.ord_of = {sid: i for i, sid in enumerate(bundle.shape_ids)}
        self.runner = eg.ScoreRunner()
        # SMs the F-IF scan leaves to other batches' kernels (query_many sets
        # it while several batches are in flight)
        self.reserve_sms = 0
        self.mode = mt.sim_mode(cfg.similarity)
        self._graphs = {}  # graph_for: captured pipelines per (stream, shape, ...)

    def scores(self, Qa, Qb=None, vq=None, vqb=None, stream=None, scan_events=None, ma=None):
        ma = self.cfg.ma if ma is None else ma
        sa = self.runner.score(self.fa, Qa, ma, self.mode, self.cfg.sigma, vq=vq,
                               stream=stream, scan_events=scan_events,
                               reserve_sms=self.reserve_sms)
        if Qb is None and self.dup:
            return sa, sa
        sb = self.runner.score(self.fb, Qa if Qb is None else Qb, ma, self.mode,
                               self.cfg.sigma, vq=vq if vqb is None else vqb, stream=stream,
                               reserve_sms=self.reserve_sms)
        return sa, sb

    def graph_for(self, stream, Q_example, top_k, rerank=True) -> "GraphedQuery":
        """The CUDA graph of this engine's pipeline on `stream` for batches
        shaped like Q_example (captured on first use, kept)."""
        key = (stream.cuda_stream, tuple(Q_example.shape), int(top_k), bool(rerank),
               int(self.reserve_sms))
        g = self._graphs.get(key)
        if g is None:
            g = self._graphs[key] = GraphedQuery(self, Q_example, top_k, rerank, stream)
        return g

    def rerank(self, sa, sb, stream=None):
        """index.py:249-258 for a batch of channel scores -> dense f64."""
        return self.sif.query(self.rerank_act(sa, sb, stream), stream=stream)

    def rerank_act(self, sa, sb, stream=None) -> eg.ActRows:
        """The query-time context activation of rerank_scores (index.py:249-256)."""
        k2 = min(self.cfg.k2, self.n)
        na, _ = eg.topk_rows(sa, k2, positive_only=True, stream=stream)
        nb = na if sb is sa else eg.topk_rows(sb, k2, positive_only=True, stream=stream)[0]
        fa = eg.act_mean(self.raw_a, nb, stream=stream)
        if sb is sa and self.raw_dup:
            final = fa  # aggregate(f, f) == f exactly (rerank.py:142-146)
        else:
            fb = eg.act_mean(self.raw_b, na, stream=stream)
            final = eg.act_aggregate(fa, fb, self.cfg.alpha, stream=stream)
        return final

    def run(self, Qa, Qb=None, top_k=10, rerank=True, self_local=None, vq=None, vqb=None,
            stream=None, scan_events=None, exact=False):
        torch.cuda.nvtx.range_push("gift.query_batch")  # timeline marker (nsys / CUPTI)
        try:
            return self._run(Qa, Qb, top_k, rerank, self_local, vq, vqb, stream, scan_events,
                             exact)
        finally:
            torch.cuda.nvtx.range_pop()

    def _run(self, Qa, Qb=None, top_k=10, rerank=True, self_local=None, vq=None, vqb=None,
             stream=None, scan_events=None, exact=False):
        """Device batch -> (idx [B, k] i32 global ordinals, val [B, k] f64).
        exact: every query view probes every cell (ma = K), which is the
        reference's exact set similarity (index.py:230-243, matching.py:55-61:
        mean over the query views of the best match over all target views;
        the ma = K degeneracy of test_matching.py:127-140)."""
        if exact:
            sa, sb = self.scores(Qa, Qb, vq, vqb, stream, scan_events, ma=self.fa.cb.K)
            if rerank:
                return self._sif_rank(self.rerank_act(sa, sb, stream), top_k, self_local, stream)
            final = sa if sb is sa else (sa + sb) / 2.0
            return eg.topk_rows(final, min(top_k, self.n), idrank=self.idrank,
                                self_local=self_local, stream=stream)
        if rerank and Qb is None and self.dup and self.raw_dup and self.cfg.k2 <= CAND_K_MAX:
            # single-channel fast path: the reduce emits per-range top-k2
            # candidates, merged into the neighbour lists (rerank.py:78-87)
            k2 = min(self.cfg.k2, self.n)
            _, cs, ci = self.runner.score(self.fa, Qa, self.cfg.ma, self.mode, self.cfg.sigma,
                                          vq=vq, stream=stream, scan_events=scan_events,
                                          cand_k=k2, dense=False,
                                          reserve_sms=self.reserve_sms)
            nbr, _ = eg.topk_candidates(cs, ci, k2, positive_only=True, stream=stream)
            fa = eg.act_mean(self.raw_a, nbr, stream=stream)
            return self._sif_rank(fa, top_k, self_local, stream)
        sa, sb = self.scores(Qa, Qb, vq, vqb, stream, scan_events)
        if rerank:
            return self._sif_rank(self.rerank_act(sa, sb, stream), top_k, self_local, stream)
        if sb is sa:
            final = sa  # np.mean([s, s], axis=0) == s exactly
        else:
            final = (sa + sb) / 2.0
        k = min(top_k, self.n)
        return eg.topk_rows(final, k, idrank=self.idrank, self_local=self_local, stream=stream)

    def rerank_lists(self, q_idx, q_val, top_k=10, self_local=None, stream=None):
        """Re-rank from given best-first F-IF neighbour lists (config 5):
        neighbours = the first k2 positive entries (top_neighbors,
        rerank.py:78-87), query activation = their raw activations' mean,
        S-IF Jaccard, final top-k (index.py:249-299)."""
        k2 = min(self.cfg.k2, q_idx.shape[1])
        nbr = torch.where(q_val[:, :k2] > 0, q_idx[:, :k2],
                          torch.full_like(q_idx[:, :k2], -1)).to(torch.int32).contiguous()
        fa = eg.act_mean(self.raw_a, nbr, stream=stream)
        return self._sif_rank(fa, top_k, self_local, stream)

    def _sif_rank(self, q: eg.ActRows, top_k, self_local=None, stream=None):
        """S-IF query + final ranking (index.py:290-299): sparse over the
        touched shapes for k <= 256, else the dense row + top-k."""
        k = min(top_k, self.n)
        if k <= 256:
            return self.sif.query_topk(q, k, self.order, self.idrank, self_local, stream=stream)
        final = self.sif.query(q, stream=stream)
        return eg.topk_rows(final, k, idrank=self.idrank, self_local=self_local, stream=stream)

    def results(self, idx_row, val_row):
        ids, labels = self.b.shape_ids, self.b.labels
        return [(ids[int(i)], float(v), labels.get(ids[int(i)], ""))
                for i, v in zip(idx_row, val_row) if i >= 0]


# ------------------------------------------------------------------ build
def _to_device_views(views, dtype):
    if torch.is_tensor(views):
        t = views
    else:
        t = torch.from_numpy(np.ascontiguousarray(views, dtype=np.float32))
    if t.dim() != 3:
        raise ValueError("views must be [n_shapes, n_views, d]")
    return t.to(nat.device()).to(dtype).contiguous()


def _self_join(fif: eg.DeviceFif, X, cfg: IndexConfig, runner: eg.ScoreRunner,
               batch: int, n: int | None = None, chunk: int = 0):
    """index.py:196-210: every database shape queried against the F-IF ->
    raw top-k1 activations and top-k2 neighbour lists (device).  X is the
    device views [n, V, d] or a provider(s0, s1) of them (streamed build)."""
    provider = X if callable(X) else None
    if n is None:
        n = X.shape[0]
    dev = fif.device
    k1 = min(cfg.k1, n)
    kk = max(k1, min(cfg.k2, n))
    raw = eg.ActRows.empty(n, max(k1, 1), dev)
    nbr = torch.full((n, max(min(cfg.k2, n), 1)), -1, dtype=torch.int32, device=dev)
    mode = mt.sim_mode(cfg.similarity)
    step = max(chunk, batch) if provider is not None else n
    for c0 in range(0, n, step):
        c1 = min(n, c0 + step)
        Xc = provider(c0, c1) if provider is not None else X
        off = c0 if provider is not None else 0
        for b0 in range(c0, c1, batch):
            b1 = min(c1, b0 + batch)
            Q = Xc[b0 - off:b1 - off].float()
            s = runner.score(fif, Q, cfg.ma, mode, cfg.sigma)
            tidx, tval = eg.topk_rows(s, kk, positive_only=True)
            eg.act_from_topk(tidx, tval, k1, out=raw.rows(b0, b1))
            nbr[b0:b1] = tidx[:, : nbr.shape[1]]
        del Xc
    return raw, nbr


def build_index_streamed(provider, shape_ids, n_views: int, dim: int,
                         config: IndexConfig = IndexConfig(), *, codebooks, labels=None,
                         chunk: int = 512, keep_features: bool = False,
                         self_join_batch: int = 256) -> IndexBundle:
    """Build from a database streamed in chunks of shapes (new; configs whose
    features do not fit HBM twice): `provider(s0, s1)`
    returns the device views [s1 - s0, n_views, dim] of shapes s0..s1 and is
    called three times per chunk (quantize, scatter, self-join), so it must be
    deterministic.  One feature set feeds both channels (D4).  Without
    keep_features the F-IF holds only the tensor-core planes (22 significant
    bits); the storage copy, `entry_features` and `save_fif` are then
    unavailable (Unsupported)."""
    shape_ids = list(shape_ids)
    if not shape_ids:
        raise EmptyManifest("no shapes listed")
    n = len(shape_ids)
    ca = codebooks["A"]
    dfa = eg.DeviceFif.build_streamed(provider, n, n_views, dim, ca.device(),
                                      dtype=config.torch_storage, chunk=chunk,
                                      keep_features=keep_features)
    fa = mt.FirstInvertedFile(ca, shape_ids, n_views, dfa)
    runner = eg.ScoreRunner()
    raw, nbr = _self_join(dfa, provider, config, runner, self_join_batch, n=n, chunk=chunk)
    final = eg.act_mean(raw, nbr)  # co_augment with one channel (rerank.py:114-125)
    sif = rr.SecondInvertedFile(shape_ids, eg.DeviceSif.build(final, n))
    acts = rr.ActivationList(raw, shape_ids)
    config = replace(config, n_views=max(1, n_views), codebook_size=ca.k)
    return IndexBundle(config=config, shape_ids=shape_ids,
                       labels=dict(labels) if labels else {s: "" for s in shape_ids},
                       codebooks={"A": ca, "B": cb.Codebook(ca.centroids, "B", ca.seed)},
                       fifs={"A": fa, "B": fa}, raw_activations={"A": acts, "B": acts}, sif=sif)


def build_index_from_views(views_a, shape_ids, config: IndexConfig = IndexConfig(), *,
                           views_b=None, labels=None, codebooks=None,
                           self_join_batch: int = 256) -> IndexBundle:
    """Build the full index from feature tensors [N, V, d] (host array or
    device tensor).  views_b=None feeds one feature set to both channels
    (computed once).  `codebooks` = {"A": Codebook, "B": ...};
    default: seeded sampled DB rows (D3)."""
    shape_ids = list(shape_ids)
    if not shape_ids:
        raise EmptyManifest("no shapes listed")
    Xa = _to_device_views(views_a, config.torch_storage)
    if Xa.shape[0] != len(shape_ids):
        raise ValueError("views and shape_ids disagree on the number of shapes")
    Xb = None if views_b is None else _to_device_views(views_b, config.torch_storage)
    if codebooks is None:
        ca = cb.sample_codebook(Xa.float().cpu().numpy(), config.codebook_size, config.seed, "A")
        cbb = (cb.Codebook(ca.centroids, "B", config.seed) if Xb is None else
               cb.sample_codebook(Xb.float().cpu().numpy(), config.codebook_size, config.seed, "B"))
        codebooks = {"A": ca, "B": cbb}
    fa = mt.build_fif_from_tensor(Xa, codebooks["A"], shape_ids)
    if Xb is None and np.array_equal(codebooks["A"].centroids, codebooks["B"].centroids):
        fb = fa
    else:
        fb = mt.build_fif_from_tensor(Xa if Xb is None else Xb, codebooks["B"], shape_ids)
    runner = eg.ScoreRunner()
    raw_a, nbr_a = _self_join(fa.dev, Xa, config, runner, self_join_batch)
    if fb is fa:
        raw_b, nbr_b = raw_a, nbr_a
    else:
        raw_b, nbr_b = _self_join(fb.dev, Xa if Xb is None else Xb, config, runner,
                                  self_join_batch)
    # co-augment (rerank.py:114-125) + aggregate (index.py:214-217)
    aug_a = eg.act_mean(raw_a, nbr_b)
    if fb is fa:
        final = aug_a
    else:
        aug_b = eg.act_mean(raw_b, nbr_a)
        final = eg.act_aggregate(aug_a, aug_b, config.alpha)
    sif = rr.SecondInvertedFile(shape_ids, eg.DeviceSif.build(final, len(shape_ids)))
    acts_a = rr.ActivationList(raw_a, shape_ids)
    acts_b = acts_a if raw_b is raw_a else rr.ActivationList(raw_b, shape_ids)
    config = replace(config, n_views=max(1, Xa.shape[1]), codebook_size=codebooks["A"].k)
    return IndexBundle(config=config, shape_ids=shape_ids,
                       labels=dict(labels) if labels else {s: "" for s in shape_ids},
                       codebooks=dict(codebooks), fifs={"A": fa, "B": fb},
                       raw_activations={"A": acts_a, "B": acts_b}, sif=sif)


def build_index_from_lists(list_idx, list_scores, shape_ids, config: IndexConfig = IndexConfig(),
                           labels=None) -> IndexBundle:
    """Config 5 (re-rank dominated): the F-IF stage is given as best-first
    neighbour lists per shape (idx [N, L] int, scores [N, L] f64, ordered by
    (score desc, ordinal asc) like build_activation's lexsort).  Raw
    activations = the first k1 positive entries (rerank.py:64-75),
    neighbourhoods = the first k2 (rerank.py:78-87), then co-augment and the
    S-IF as in index.py:211-218.  The bundle has no F-IF (query with
    `QueryEngine.rerank_lists`)."""
    shape_ids = list(shape_ids)
    dev = nat.device()
    idx = torch.as_tensor(list_idx).to(dev, dtype=torch.int32).contiguous()
    val = torch.as_tensor(list_scores).to(dev, dtype=torch.float64).contiguous()
    n, L = idx.shape
    if n != len(shape_ids):
        raise ValueError("lists and shape_ids disagree on the number of shapes")
    k1, k2 = min(config.k1, L), min(config.k2, L)
    srt = torch.sort(idx, dim=1).values  # a score row lists each shape once (rerank.py:64-75)
    if bool(((srt[:, 1:] == srt[:, :-1]) & (srt[:, 1:] >= 0)).any()):
        raise ValueError("neighbour lists must not repeat a shape within a row")
    del srt
    raw = eg.act_from_topk(idx, val, k1)
    nbr = torch.where(val[:, :k2] > 0, idx[:, :k2], torch.full_like(idx[:, :k2], -1)).contiguous()
    final = eg.act_mean(raw, nbr)
    sif = rr.SecondInvertedFile(shape_ids, eg.DeviceSif.build(final, n))
    acts = rr.ActivationList(raw, shape_ids)
    return IndexBundle(config=config, shape_ids=shape_ids,
                       labels=dict(labels) if labels else {s: "" for s in shape_ids},
                       codebooks={}, fifs={"A": None, "B": None},
                       raw_activations={"A": acts, "B": acts}, sif=sif)


def build_index(manifest, config: IndexConfig = IndexConfig(), jobs: int = 1,
                feature_files: dict | None = None, codebooks=None) -> IndexBundle:
    """index.py:146-227 from precomputed feature files ({"A": path, "B":
    path}); mesh rendering (index.py:106-139) is outside the GPU path.
    Without `codebooks` each channel's codebook is trained like the
    reference's (k-means over the non-zero views, codebook_size, seed) by
    `codebook.train_codebook` on the device."""
    if isinstance(manifest, (str, Path)):
        rows = read_manifest(manifest)
    else:
        rows = [(Path(p), lab) for p, lab in manifest]
    if not rows:
        raise EmptyManifest("no shapes listed")
    if not feature_files:
        return _build_index_rendered(rows, config, jobs, codebooks)
    if set(feature_files) != set(CHANNELS):
        raise ChannelMismatch(f"feature files required for channels {CHANNELS}")
    config = replace(config, imported=True)
    # device ingest (features.FeatureFile): rows stream from the files to the
    # GPU and are re-normalized there, bit-identical to import_features
    ffs = {ch: ft.FeatureFile(feature_files[ch], ch) for ch in CHANNELS}
    sel = {ch: [] for ch in CHANNELS}
    ids, labels = [], {}
    for path, label in rows:
        sid = Path(path).stem
        if sid not in ffs["A"]._index or sid not in ffs["B"]._index:
            log.warning("skipping shape %s: not present in feature files", sid)
            continue
        ids.append(sid)
        labels[sid] = label
        for ch in CHANNELS:
            sel[ch].append(ffs[ch].index_of(sid))
    if not ids:
        raise AllShapesFailed("every shape in the manifest failed to build")
    va = ffs["A"].device_rows(sel["A"])
    if (os.path.realpath(ffs["A"].path) == os.path.realpath(ffs["B"].path)
            and sel["A"] == sel["B"]):
        vb = None  # one feature set feeds both channels (D4)
    else:
        vb = ffs["B"].device_rows(sel["B"])
        if vb.shape == va.shape and torch.equal(va, vb):
            vb = None
    if codebooks is None:
        codebooks = _train_codebooks(va, vb, config)
    return build_index_from_views(va, ids, config, views_b=vb, labels=labels,
                                  codebooks=codebooks)


def _train_codebooks(va, vb, config):
    """index.py:186-193: k-means per channel over the non-zero views, on the
    device (channel B reuses A's centroids when the features are the same)."""
    codebooks = {}
    for ch, v in (("A", va), ("B", va if vb is None else vb)):
        if ch == "B" and vb is None:
            codebooks["B"] = cb.Codebook(codebooks["A"].centroids, "B", config.seed)
            continue
        rows = v.reshape(-1, v.shape[-1])
        codebooks[ch] = cb.train_codebook(rows[rows.any(dim=1)], k=config.codebook_size,
                                          seed=config.seed, channel=ch)
    return codebooks


def _build_index_rendered(rows, config, jobs, codebooks):
    """index.py:146-227 from meshes: the plugged-in CPU renderer gives the
    view sets (`set_renderer`), everything after them runs on the device."""
    if _Renderer.compute_viewset is None:
        raise Unsupported("mesh rendering is outside the GPU path: pass feature_files, use "
                          "build_index_from_views, or plug a renderer (set_renderer)")
    built = _gather_viewsets(rows, config, jobs)
    if not built:
        raise AllShapesFailed("every shape in the manifest failed to build")
    ids = [vs.shape_id for _row, vs in built]
    labels = {vs.shape_id: row[1] for row, vs in built}
    dev = nat.device()
    va = torch.from_numpy(np.stack([vs.matrix("A") for _r, vs in built]).astype(np.float32))
    vb = torch.from_numpy(np.stack([vs.matrix("B") for _r, vs in built]).astype(np.float32))
    va, vb = va.to(dev), vb.to(dev)
    if codebooks is None:
        codebooks = _train_codebooks(va, vb, config)
    return build_index_from_views(va, ids, config, views_b=vb, labels=labels,
                                  codebooks=codebooks)


def build_index_from_feature_file(path, config: IndexConfig = IndexConfig(), *, codebooks,
                                  labels=None, chunk: int = 512, self_join_batch: int = 256,
                                  keep_features: bool = False) -> IndexBundle:
    """One GIFTFT1 file feeding both channels (D4), streamed through the
    chunked build (`build_index_streamed`): shapes are read from the file,
    normalized on the GPU and consumed chunk by chunk, so the database never
    sits in host memory (SURVEY.md §8(f) row 2, config-3 scale)."""
    f = ft.FeatureFile(path, "A")
    if not len(f):
        raise EmptyManifest(f"feature file {path} lists no shapes")
    config = replace(config, imported=True)
    return build_index_streamed(f.provider(), f.shape_ids, f.n_views, f.dim, config,
                                codebooks=codebooks, labels=labels, chunk=chunk,
                                keep_features=keep_features, self_join_batch=self_join_batch)


# ------------------------------------------------------------------ query
def _viewset_mats(bundle, target):
    if isinstance(target, ft.ViewSet):
        try:
            ma_ = target.matrix("A")
            mb_ = target.matrix("B")
        except KeyError as exc:
            raise ChannelMismatch(f"query lacks channel {exc.args[0]!r}") from exc
        return ma_, mb_, target.shape_id
    if isinstance(target, np.ndarray) or torch.is_tensor(target):
        return target, target, ""
    raise ChannelMismatch("queries must be view sets or feature matrices "
                          "(mesh rendering is outside the GPU path)")


def query(bundle: IndexBundle, target, top_k: int = 10, exact: bool = False,
          rerank: bool = True):
    """Rank database shapes for one query view set (index.py:261-299).
    Returns ([(shape_id, score, label)], {"render": s, "match": s})."""
    if bundle.n_shapes == 0:
        raise EmptyIndex("index holds no shapes")
    eng = bundle.engine
    if exact and eng.fa is None:
        raise Unsupported("exact ranking needs the stored view features (F-IF)")
    render_s = 0.0
    if _Renderer.mesh_type is not None and isinstance(target, _Renderer.mesh_type):
        if bundle.config.imported:  # index.py:273-275
            raise ChannelMismatch("index was built from imported features; query by id instead")
        t0 = time.perf_counter()
        target = _Renderer.compute_viewset(target, bundle.config)
        render_s = time.perf_counter() - t0
    ma_, mb_, sid = _viewset_mats(bundle, target)
    t0 = time.perf_counter()
    qa = mt._as_query_tensor(ma_, bundle.fifs["A"].dim)[None]
    qb = None
    if not (eng.dup and (mb_ is ma_ or np.array_equal(np.asarray(ma_), np.asarray(mb_)))):
        qb = mt._as_query_tensor(mb_, bundle.fifs["B"].dim)[None]
    self_local = torch.tensor([eng.ord_of.get(sid, -1)], dtype=torch.int32, device=qa.device)
    idx, val = eng.run(qa, qb, top_k=top_k, rerank=rerank, self_local=self_local, exact=exact)
    idx, val = idx.cpu().numpy(), val.cpu().numpy()
    t1 = time.perf_counter()
    return eng.results(idx[0], val[0]), {"render": render_s, "match": t1 - t0}


def query_by_id(bundle: IndexBundle, shape_id: str, top_k: int = 10, exact: bool = False,
                rerank: bool = True):
    """Query with a database shape's stored views, recovered cell-major with
    zero views absent (index.py:302-314)."""
    if shape_id not in bundle.engine.ord_of:
        raise EmptyIndex(f"unknown shape id {shape_id!r}")
    o = bundle.engine.ord_of[shape_id]
    vs = ft.ViewSet(shape_id=shape_id)
    for ch in CHANNELS:
        mat = bundle.viewset_matrix(ch, o)
        vs.descriptors[ch] = [ft.ViewDescriptor(values=row.astype(np.float32), channel=ch)
                              for row in mat]
    return query(bundle, vs, top_k=top_k, exact=exact, rerank=rerank)


def rerank_scores(bundle: IndexBundle, channel_scores: dict) -> np.ndarray:
    """Contextual re-ranked similarity from per-channel match scores
    (index.py:249-258)."""
    dev = nat.device()
    sa = torch.from_numpy(np.asarray(channel_scores["A"], dtype=np.float64)[None].copy()).to(dev)
    if np.array_equal(channel_scores["A"], channel_scores["B"]):
        sb = sa
    else:
        sb = torch.from_numpy(np.asarray(channel_scores["B"], dtype=np.float64)[None].copy()).to(dev)
    return bundle.engine.rerank(sa, sb)[0].cpu().numpy()


def query_batch(bundle: IndexBundle, views, top_k: int = 10, rerank: bool = True,
                self_ids=None, views_b=None):
    """Batched `query` (new): views [B, V, d] (host or device) -> list of
    result lists, identical to calling `query` on each view set."""
    eng = bundle.engine
    Qa = views if torch.is_tensor(views) else torch.from_numpy(np.ascontiguousarray(views, np.float32))
    Qa = Qa.to(nat.device(), dtype=torch.float32)
    Qb = None
    if views_b is not None:
        Qb = views_b if torch.is_tensor(views_b) else torch.from_numpy(
            np.ascontiguousarray(views_b, np.float32))
        Qb = Qb.to(nat.device(), dtype=torch.float32)
    B = Qa.shape[0]
    selfs = [eng.ord_of.get(s, -1) for s in (self_ids or [""] * B)]
    self_local = torch.tensor(selfs, dtype=torch.int32, device=Qa.device)
    out = []
    bs = bundle.config.batch_size
    for b0 in range(0, B, bs):
        b1 = min(B, b0 + bs)
        idx, val = eng.run(Qa[b0:b1], None if Qb is None else Qb[b0:b1], top_k=top_k,
                           rerank=rerank, self_local=self_local[b0:b1])
        idx, val = idx.cpu().numpy(), val.cpu().numpy()
        out.extend(eng.results(i, v) for i, v in zip(idx, val))
    return out


_LANES: dict = {}
LANE_RESERVE_SMS = 44  # config 2, 4 lanes, 3 runs each: 0 SMs ~40.6k, 20 41.2k, 28 41.9k, 36-64 42.2-42.5k q/s


_PINNED = threading.local()


def _pinned(tag: str, n: int, dtype) -> torch.Tensor:
    """A grow-only pinned host buffer of at least n elements, kept per tag in
    the calling thread (released with the thread)."""
    bufs = getattr(_PINNED, "bufs", None)
    if bufs is None:
        bufs = _PINNED.bufs = {}
    buf = bufs.get(tag)
    if buf is None or buf.numel() < n or buf.dtype != dtype:
        buf = bufs[tag] = torch.empty(max(n, 1), dtype=dtype, pin_memory=True)
    return buf[:n]


def lane_streams(n: int) -> list:
    """The first n persistent side streams of the current device (scratch
    buffers are kept per stream, so reusing the streams reuses them)."""
    dev = torch.cuda.current_device()
    have = _LANES.setdefault(dev, [])
    while len(have) < n:
        have.append(torch.cuda.Stream(device=dev))
    return have[:n]


class GraphedQuery:
    """One query batch's whole device pipeline (QueryEngine.run: quantize,
    plan, scan, reduce, neighbours, S-IF, ranking -- ~40 kernels) captured
    once in a CUDA graph on `stream` over a static [B, V, d] input buffer and
    replayed per batch: one launch instead of ~40 (configs 1-2 issue faster
    than Python launches them).  Every kernel of the path is graph-safe: the
    plan's sizes live on the device, nothing synchronises with the host.
    Calling it copies Q into the buffer and replays on `stream`; the returned
    (idx, val) are the graph's static outputs, overwritten by the next call.
    Results are identical to eng.run (tested)."""

    def __init__(self, eng, Q_example: torch.Tensor, top_k: int, rerank: bool = True,
                 stream=None):
        self.stream = stream if stream is not None else torch.cuda.Stream()
        self.q = torch.empty_like(Q_example)
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            self.q.copy_(Q_example)
            for _ in range(2):  # eager warm-up: workspaces, scratch and cached sizes
                eng.run(self.q, top_k=top_k, rerank=rerank)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.out = eng.run(self.q, top_k=top_k, rerank=rerank)
        self.stream.synchronize()

    def __call__(self, Q: torch.Tensor):
        with torch.cuda.stream(self.stream):
            self.q.copy_(Q, non_blocking=True)
            self.graph.replay()
        return self.out


def query_many(bundle: IndexBundle, views_host: torch.Tensor, top_k: int = 10,
               rerank: bool = True, batch_size: int | None = None, lanes: int = 2,
               reserve_sms: int | None = None, graph: bool = False):
    """Throughput API (new): queries from pinned host memory [Q, V, d] f32,
    processed in device batches on `lanes` compute streams, the host->device
    copy of the next batches overlapped with the compute on a copy stream.
    With lanes > 1 the scan leaves `reserve_sms` SMs (default
    LANE_RESERVE_SMS) to the other batches' kernels, which cannot share an SM
    with a scan CTA (shared memory / TMEM).  graph: full batches replay a
    CUDA graph of the pipeline per lane (`GraphedQuery`, captured on first
    use and kept on the engine).  Returns host (idx [Q, k] int32 global
    ordinals, val [Q, k] f64)."""
    eng = bundle.engine
    bs = batch_size or bundle.config.batch_size
    Qn, V, d = views_host.shape
    k = min(top_k, eng.n)
    dev = nat.device()
    main = torch.cuda.current_stream()
    L = max(1, int(lanes))
    # batch i computes on lane i % L (its own stream and scratch), so one
    # batch's quantize / reduce / re-rank kernels overlap the other's scan
    # side streams only: the legacy default stream would serialize with the copies
    comp = lane_streams(L)
    copy = lane_streams(L + 1)[L]
    # input buffers: batch i lands in buffer i % NB; one more than the lanes,
    # so the next batch's copy runs while every lane computes (config 3:
    # 268 MB per batch, 5 ms of PCIe)
    NB = L + 1
    bufs = [torch.empty((bs, V, d), dtype=torch.float32, device=dev) for _ in range(NB)]
    ready = [torch.cuda.Event() for _ in range(NB)]
    free = [torch.cuda.Event() for _ in range(NB)]
    # pinned result buffers are kept between calls (a pinned allocation is a
    # host-blocking driver call of ~0.1-1 ms: config 1's whole batch time);
    # the caller gets copies
    out_idx = _pinned("idx", Qn * k, torch.int32).view(Qn, k)
    out_val = _pinned("val", Qn * k, torch.float64).view(Qn, k)
    nb = (Qn + bs - 1) // bs

    def issue(i):
        s = i % NB
        b0, b1 = i * bs, min(Qn, (i + 1) * bs)
        with torch.cuda.stream(copy):
            copy.wait_event(free[s])
            bufs[s][: b1 - b0].copy_(views_host[b0:b1], non_blocking=True)
            ready[s].record(copy)

    prev_reserve = eng.reserve_sms
    if reserve_sms is None:
        reserve_sms = LANE_RESERVE_SMS if L > 1 else 0
    eng.reserve_sms = reserve_sms
    for c in comp:
        c.wait_stream(main)
    for s in range(NB):
        free[s].record(main)
    for i in range(min(NB, nb)):
        issue(i)
    for i in range(nb):
        s = i % NB
        b0, b1 = i * bs, min(Qn, (i + 1) * bs)
        cs = comp[i % L]
        with torch.cuda.stream(cs):
            cs.wait_event(ready[s])
            if graph and b1 - b0 == bs:
                gq = eng.graph_for(cs, bufs[s], k, rerank)
                idx, val = gq(bufs[s])  # copies the batch into the graph's input
            else:
                idx, val = eng.run(bufs[s][: b1 - b0], top_k=k, rerank=rerank)
            free[s].record(cs)
            out_idx[b0:b1].copy_(idx, non_blocking=True)
            out_val[b0:b1].copy_(val, non_blocking=True)
        if i + NB < nb:
            issue(i + NB)
    for c in comp:
        main.wait_stream(c)
    eng.reserve_sms = prev_reserve
    main.synchronize()
    return out_idx.numpy().copy(), out_val.numpy().copy()


# ------------------------------------------------------------------ evaluation
def _eval_ranks(eng, final: torch.Tensor, rows: torch.Tensor, rel_host: list) -> list:
    """Ranks of each query's relevant shapes in its ranking (key: score desc,
    shape id asc; the query itself excluded) -- libgift gift_eval_ranks."""
    B = final.shape[0]
    R = max(1, max(len(r) for r in rel_host))
    rel = np.full((B, R), -1, dtype=np.int32)
    for b, r in enumerate(rel_host):
        rel[b, :len(r)] = r
    rel_d = torch.from_numpy(rel).to(final.device)
    out = torch.empty((B, R), dtype=torch.int32, device=final.device)
    nat.call("gift_eval_ranks", nat.ptr(final.contiguous()), B, final.shape[1],
             nat.ptr(eng.idrank), nat.ptr(rows.to(torch.int32).contiguous()), nat.ptr(rel_d), R,
             nat.ptr(out), nat.stream_ptr())
    ranks = out.cpu().numpy()
    return [np.sort(ranks[b, :len(r)]) for b, r in enumerate(rel_host)]


def _labelled_queries(bundle):
    """index.py:320-327: class sizes; shapes of classes with >= 2 members are
    queries, the others are skipped; relevant shapes = same class, not self."""
    ids, labels = bundle.shape_ids, bundle.labels
    lab = [labels.get(s, "") for s in ids]
    groups = {}
    for i, x in enumerate(lab):
        groups.setdefault(x, []).append(i)
    sizes = {x: len(g) for x, g in groups.items()}
    keep = [i for i in range(len(ids)) if sizes[lab[i]] >= 2]
    return lab, groups, sizes, keep, len(ids) - len(keep)


def _device_report(bundle, scores_of, batch_size=None):
    from . import evaluation as ev

    eng = bundle.engine
    lab, groups, sizes, keep, skipped = _labelled_queries(bundle)
    dev = nat.device()
    bs = batch_size or bundle.config.batch_size
    per_query = []
    for b0 in range(0, len(keep), bs):
        sel = keep[b0:b0 + bs]
        rows = torch.tensor(sel, dtype=torch.int64, device=dev)
        final = scores_of(rows)
        rel = [[j for j in groups[lab[i]] if j != i] for i in sel]
        for i, ranks in zip(sel, _eval_ranks(eng, final, rows, rel)):
            per_query.append(ev.metrics_from_ranks(ranks, sizes[lab[i]], lab[i]))
    return ev.aggregate_report(per_query, n_skipped=skipped)


def evaluate_index(bundle: IndexBundle, exact: bool = False, rerank: bool = True,
                   batch_size: int | None = None):
    """Every labelled database shape (class of >= 2) queried with its stored
    views, excluded from its own ranking, scored (index.py:317-333).  The
    queries run through the device pipeline in batches; each query's ranking
    (score desc, shape id asc) is resolved on the device as the 1-based ranks
    of its relevant shapes (gift_eval_ranks)."""
    eng = bundle.engine
    if eng.fa is None:
        raise Unsupported("evaluation needs the stored view features (F-IF)")

    def scores_of(rows):
        Q, vq = eng.fa.shape_views(rows)  # query_by_id: stored views, cell-major
        Qb = vqb = None
        if not eng.dup:  # channel B's own stored views (its own dimension)
            Qb, vqb = eng.fb.shape_views(rows)
        sa, sb = eng.scores(Q, Qb, vq=vq, vqb=vqb, ma=eng.fa.cb.K if exact else None)
        return eng.rerank(sa, sb) if rerank else (sa if sb is sa else (sa + sb) / 2.0)

    return _device_report(bundle, scores_of, batch_size)


def exact_baseline_report(bundle: IndexBundle, channel: str = "B", variant: str = "robust",
                          batch_size: int | None = None):
    """Single-channel exact ranking over the database, scored (index.py:
    336-357): each labelled shape's stored views of `channel` against every
    shape's by exact_similarity (the scan with every view probing every cell:
    mean over the query views of the best clamped cosine), ranked by (score
    desc, id asc) without the query itself.  `variant` is accepted and, as in
    the reference, does not change the similarity used."""
    eng = bundle.engine
    if channel not in CHANNELS:
        raise ChannelMismatch(f"unknown channel {channel!r}")
    fif = eng.fa if channel == "A" else eng.fb
    if fif is None:
        raise Unsupported("the exact baseline needs the stored view features (F-IF)")

    def scores_of(rows):
        Q, vq = fif.shape_views(rows)
        return eng.runner.score(fif, Q, fif.cb.K, nat.SIM_COSINE, 0.5, vq=vq)

    return _device_report(bundle, scores_of, batch_size)


# ------------------------------------------------------------------ persistence
def save_bundle(bundle: IndexBundle, out_dir) -> Path:
    """Versioned directory with deterministic bytes (index.py:360-375)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    cfg = asdict(bundle.config)
    defaults = IndexConfig()
    extra = {k: v for k, v in cfg.items()
             if k not in _REFERENCE_FIELDS and getattr(defaults, k) != v}
    meta = {"version": bundle.version,
            "config": {k: cfg[k] for k in _REFERENCE_FIELDS} | extra}
    with open(out / "config.json", "w", encoding="utf-8") as fh:
        json.dump(meta, fh, indent=2, sort_keys=True)
        fh.write("\n")
    with open(out / "shapes.tsv", "w", encoding="utf-8", newline="\n") as fh:
        for sid in bundle.shape_ids:
            fh.write(f"{sid}\t{bundle.labels.get(sid, '')}\n")
    for ch in CHANNELS:
        cb.save_codebook(bundle.codebooks[ch], out / f"codebook_{ch}.bin")
        mt.save_fif(bundle.fifs[ch], out / f"fif_{ch}.bin")
        rr.save_activations(bundle.raw_activations[ch], out / f"activations_{ch}.bin")
    rr.save_sif(bundle.sif, out / "sif.bin")
    return out


def load_bundle(index_dir) -> IndexBundle:
    """index.py:378-414; identical channel files are loaded once."""
    index_dir = Path(index_dir)
    try:
        with open(index_dir / "config.json", encoding="utf-8") as fh:
            meta = json.load(fh)
    except FileNotFoundError as exc:
        raise FormatError(f"no index bundle at {index_dir}") from exc
    if meta.get("version") != FORMAT_VERSION:
        raise FormatError(f"unsupported index version {meta.get('version')!r}")
    known = {f.name for f in fields(IndexConfig)}
    config = IndexConfig(**{k: v for k, v in meta["config"].items() if k in known})
    ids, labels = [], {}
    for line in (index_dir / "shapes.tsv").read_text(encoding="utf-8").splitlines():
        if not line:
            continue
        sid, _, label = line.partition("\t")
        ids.append(sid)
        labels[sid] = label
    raw_bytes = {ch: (index_dir / f"fif_{ch}.bin").read_bytes() for ch in CHANNELS}
    cbs, fifs, acts = {}, {}, {}
    for ch in CHANNELS:
        cbs[ch] = cb.load_codebook(index_dir / f"codebook_{ch}.bin")
    same = (raw_bytes["A"] == raw_bytes["B"]
            and np.array_equal(cbs["A"].centroids, cbs["B"].centroids))
    fifs["A"] = mt.load_fif(index_dir / "fif_A.bin", cbs["A"], config.torch_storage)
    fifs["B"] = fifs["A"] if same else mt.load_fif(index_dir / "fif_B.bin", cbs["B"],
                                                   config.torch_storage)
    act_bytes = {ch: (index_dir / f"activations_{ch}.bin").read_bytes() for ch in CHANNELS}
    for ch in CHANNELS:
        if ch == "B" and act_bytes["A"] == act_bytes["B"]:
            acts["B"] = acts["A"]
            continue
        host = rr.load_activations(index_dir / f"activations_{ch}.bin")
        cap = max([a.support for a in host] + [1])
        acts[ch] = rr.ActivationList(eg.ActRows.from_host(host, cap), [a.owner for a in host])
    sif = rr.load_sif(index_dir / "sif.bin")
    return IndexBundle(config=config, shape_ids=ids, labels=labels, codebooks=cbs, fifs=fifs,
                       raw_activations=acts, sif=sif, version=meta["version"])
