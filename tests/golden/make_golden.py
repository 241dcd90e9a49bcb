"""Generate the golden vectors under tests/golden/ by running the REFERENCE
implementation (`shapesearch`, /root/reference/pkg/src) on seeded inputs.

Run in the build container (the reference does not travel to the GPU box):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
Only reference public functions are called; the index bundle is assembled
from them the way index.build_index does (index.py:185-227) except that the
codebook is a sampled one (SURVEY.md divergence D3) and the one feature set
feeds both channels (D4).
"""

from __future__ import annotations

import io
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from cases import (E2E_CASES, EVAL_CASES, KMEANS_CASES, kmeans_inputs, mixture_views,  # noqa: E402
                   sampled_codebook, shape_ids, unit_nonneg_rows)
from shapesearch import codebook as rcb  # noqa: E402
from shapesearch import features as rft  # noqa: E402
from shapesearch import index as rix  # noqa: E402
from shapesearch import matching as rmt  # noqa: E402
from shapesearch import rerank as rrr  # noqa: E402


def as_viewset(sid, mat, channels=("A", "B")):
    vs = rft.ViewSet(shape_id=sid)
    for ch in channels:
        for row in mat:
            vs.add(ch, rft.ViewDescriptor(values=np.asarray(row, dtype=np.float32), channel=ch))
    return vs


def golden_quantize():
    rng = np.random.default_rng(2024)
    out = {}
    cases = []
    # 1. generic f64 inputs
    C = rng.random((10, 8)).astype(np.float32)
    X = rng.random((40, 8))
    cases += [(C, X, 1), (C, X, 2), (C, X, 10)]
    # 2. duplicated centroids (exact ties -> lower index) + exact centroid queries
    C2 = rng.random((9, 6)).astype(np.float32)
    C2[4] = C2[1]
    C2[7] = C2[1]
    X2 = np.concatenate([C2.astype(np.float64), rng.random((12, 6))])
    cases += [(C2, X2, 1), (C2, X2, 3), (C2, X2, 9)]
    # 3. odd dims / pairwise tree shapes
    for d, k, ma in ((5, 7, 7), (129, 12, 2), (300, 20, 3), (1000, 16, 2)):
        Cd = unit_nonneg_rows(rng, k, d)
        Xd = unit_nonneg_rows(rng, 24, d).astype(np.float64)
        cases.append((Cd, Xd, ma))
    # 4. mixture rows at d = 4096 (config 2 dimension), f32 queries
    views, _ = mixture_views(77, 40, 4, 4096, 6, mu0=-0.26)
    Cm = sampled_codebook(views, 64, 5)
    Xm = views.reshape(-1, 4096)[:96].astype(np.float64)
    cases += [(Cm, Xm, 1), (Cm, Xm, 2)]
    for i, (C, X, ma) in enumerate(cases):
        cb = rcb.Codebook(centroids=C)
        res = np.stack([rcb.quantize(cb, x, ma=ma) for x in X])
        out[f"c{i}_C"] = C
        out[f"c{i}_X"] = X
        out[f"c{i}_ma"] = np.int64(ma)
        out[f"c{i}_out"] = res.astype(np.int64)
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "quantize.npz"), **out)


def golden_fif():
    out = {}
    views, _ = mixture_views(31, 12, 6, 16, 3, zero_views=3, n_queries=4)
    db, qs = views[:12], views[12:]
    ids = shape_ids(12)
    for tag, k in (("k5", 5), ("k1", 1)):
        C = sampled_codebook(db, k, 3)
        cb = rcb.Codebook(centroids=C, channel="A")
        vsets = [as_viewset(ids[i], db[i], ("A",)) for i in range(12)]
        fif = rmt.build_fif(vsets, cb, "A")
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "fif.bin")
            rmt.save_fif(fif, path)
            out[f"{tag}_fif_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        out[f"{tag}_C"] = C
        lens = [len(o) for o in fif.entry_ordinals]
        out[f"{tag}_entry_len"] = np.array(lens, dtype=np.int64)
        out[f"{tag}_entry_ord"] = np.concatenate(fif.entry_ordinals).astype(np.int32)
        out[f"{tag}_entry_feat"] = np.concatenate(fif.entry_features).astype(np.float32)
        for ma in sorted({1, min(2, k), k}):
            sc = np.stack([rmt.query_fif(fif, q, ma=ma) for q in list(qs) + list(db[:3])])
            out[f"{tag}_scores_ma{ma}"] = sc
        out[f"{tag}_shape_matrix_0"] = fif.shape_matrix(0)
    out["db"] = db
    out["queries"] = qs
    np.savez_compressed(os.path.join(HERE, "fif.npz"), **out)


def golden_rerank():
    rng = np.random.default_rng(4242)
    out = {}
    # build_activation / top_neighbors on scores with ties and zeros
    S = np.round(rng.random((6, 30)), 2)
    S[:, rng.choice(30, 8, replace=False)] = 0.0
    S[1] = 0.0
    out["scores"] = S
    for k in (1, 4, 10, 40):
        acts = [rrr.build_activation(s, k) for s in S]
        out[f"act_k{k}_idx"] = [a.indices for a in acts] and np.concatenate([a.indices for a in acts])
        out[f"act_k{k}_len"] = np.array([a.support for a in acts])
        out[f"act_k{k}_val"] = np.concatenate([a.values for a in acts])
        out[f"act_k{k}_norm"] = np.array([a.norm for a in acts])
        nb = [rrr.top_neighbors(s, k) for s in S]
        out[f"nbr_k{k}_len"] = np.array([len(x) for x in nb])
        out[f"nbr_k{k}"] = np.array(sum(nb, []), dtype=np.int64)
    # co_augment over random activations / neighbourhoods
    n = 16
    def rand_act(owner):
        sup = rng.choice(n, size=int(rng.integers(1, 6)), replace=False)
        return rrr.make_activation(owner, sup, rng.random(len(sup)) * 0.9 + 0.1)
    a1 = [rand_act(f"a{i}") for i in range(n)]
    a2 = [rand_act(f"b{i}") for i in range(n)]
    n1 = [list(rng.choice(n, size=int(rng.integers(0, 4)), replace=False)) for _ in range(n)]
    n2 = [list(rng.choice(n, size=int(rng.integers(0, 4)), replace=False)) for _ in range(n)]
    c1, c2 = rrr.co_augment(a1, a2, n1, n2)
    def pack(prefix, acts):
        out[f"{prefix}_len"] = np.array([a.support for a in acts])
        out[f"{prefix}_idx"] = np.concatenate([a.indices for a in acts])
        out[f"{prefix}_val"] = np.concatenate([a.values for a in acts])
        out[f"{prefix}_norm"] = np.array([a.norm for a in acts])
    pack("a1", a1)
    pack("a2", a2)
    out["n1_len"] = np.array([len(x) for x in n1])
    out["n1"] = np.array(sum(n1, []), dtype=np.int64)
    out["n2_len"] = np.array([len(x) for x in n2])
    out["n2"] = np.array(sum(n2, []), dtype=np.int64)
    pack("co1", c1)
    pack("co2", c2)
    for alpha in (0.25, 0.5, 1.0, 2.0):
        pack(f"agg{alpha}", [rrr.aggregate(x, y, alpha) for x, y in zip(c1, c2)])
    sif = rrr.build_sif(c1)
    out["sif_len"] = np.array([len(o) for o in sif.entry_ordinals])
    out["sif_ord"] = np.concatenate(sif.entry_ordinals)
    out["sif_val"] = np.concatenate(sif.entry_values)
    out["sif_norms"] = sif.norms
    out["sif_scores"] = np.stack([rrr.query_sif(sif, q) for q in c1 + c2])
    np.savez_compressed(os.path.join(HERE, "rerank.npz"), **out)


def reference_bundle(db, ids, C, cfg):
    """index.py:185-227 with a given codebook; channel B = channel A."""
    vsets = [as_viewset(ids[i], db[i]) for i in range(len(ids))]
    codebooks, fifs = {}, {}
    for ch in rix.CHANNELS:
        codebooks[ch] = rcb.Codebook(centroids=C, channel=ch, seed=cfg.seed)
        fifs[ch] = rmt.build_fif(vsets, codebooks[ch], ch)
    scores = {ch: [rmt.query_fif(fifs[ch], vs.matrix(ch), ma=cfg.ma) for vs in vsets]
              for ch in rix.CHANNELS}
    raw = {ch: [rrr.build_activation(scores[ch][i], cfg.k1, owner=ids[i]) for i in range(len(ids))]
           for ch in rix.CHANNELS}
    nbr = {ch: [rrr.top_neighbors(scores[ch][i], cfg.k2) for i in range(len(ids))]
           for ch in rix.CHANNELS}
    aa, ab = rrr.co_augment(raw["A"], raw["B"], nbr["A"], nbr["B"])
    final = [rrr.aggregate(x, y, cfg.alpha) for x, y in zip(aa, ab)]
    sif = rrr.build_sif(final, shape_ids=ids)
    bundle = rix.IndexBundle(config=cfg, shape_ids=list(ids), labels={i: "" for i in ids},
                             codebooks=codebooks, fifs=fifs, raw_activations=raw, sif=sif)
    return bundle, scores, raw, nbr, final


def golden_e2e():
    for (name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv) in E2E_CASES:
        views, _ = mixture_views(seed, N, V, d, classes, zero_views=zv, n_queries=nq)
        db, qs = views[:N], views[N:]
        ids = shape_ids(N)
        C = sampled_codebook(db, K, seed + 1)
        cfg = rix.IndexConfig(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2, imported=True)
        bundle, scores, raw, nbr, final = reference_bundle(db, ids, C, cfg)
        out = {"C": C}
        out["db_scores"] = np.stack(scores["A"]) if N <= 200 else np.zeros(0)
        out["raw_len"] = np.array([a.support for a in raw["A"]])
        out["raw_idx"] = np.concatenate([a.indices for a in raw["A"]])
        out["raw_val"] = np.concatenate([a.values for a in raw["A"]])
        out["raw_norm"] = np.array([a.norm for a in raw["A"]])
        out["nbr_len"] = np.array([len(x) for x in nbr["A"]])
        out["nbr"] = np.array(sum(nbr["A"], []), dtype=np.int64)
        out["final_len"] = np.array([a.support for a in final])
        out["final_idx"] = np.concatenate([a.indices for a in final])
        out["final_val"] = np.concatenate([a.values for a in final])
        out["final_norm"] = np.array([a.norm for a in final])
        for rerank in (True, False):
            tag = "rr" if rerank else "nr"
            rid, rsc = [], []
            for q in qs:
                res, _t = rix.query(bundle, as_viewset("query", q), top_k=top_k, rerank=rerank)
                rid.append([ids.index(r[0]) for r in res])
                rsc.append([r[1] for r in res])
            out[f"q_{tag}_ids"] = np.array(rid, dtype=np.int64)
            out[f"q_{tag}_scores"] = np.array(rsc)
            bid, bsc = [], []
            for i in range(0, N, max(1, N // 8)):
                res, _t = rix.query_by_id(bundle, ids[i], top_k=top_k, rerank=rerank)
                bid.append([ids.index(r[0]) for r in res])
                bsc.append([r[1] for r in res])
            out[f"id_{tag}_ids"] = np.array(bid, dtype=np.int64)
            out[f"id_{tag}_scores"] = np.array(bsc)
        out["q_fif_scores"] = np.stack([rmt.query_fif(bundle.fifs["A"], q, ma=ma) for q in qs])
        out["q_rerank_scores"] = np.stack([
            rix.rerank_scores(bundle, {"A": s, "B": s})
            for s in out["q_fif_scores"]])
        np.savez_compressed(os.path.join(HERE, f"e2e_{name}.npz"), **out)
        print(name, "done")


def golden_c1():
    """BASELINE.json config 1 exactly (N=1,000 x V=64 x d=256, 40 classes,
    sigma 0.3, K=64 sampled centroids, ma=1, k1=10, k2=4, 100 queries,
    top-50), cosine mode, built and queried by the reference itself (both
    channels computed, as the reference does).  Inputs are regenerated from
    cases.c1_inputs() on the GPU box."""
    from cases import C1, c1_inputs

    db, qs, C, ids = c1_inputs()
    cfg = rix.IndexConfig(n_views=C1["V"], codebook_size=C1["K"], ma=C1["ma"], k1=C1["k1"],
                          k2=C1["k2"], imported=True)
    bundle, scores, raw, nbr, final = reference_bundle(db, ids, C, cfg)
    out = {"C": C}
    out["raw_len"] = np.array([a.support for a in raw["A"]])
    out["raw_idx"] = np.concatenate([a.indices for a in raw["A"]])
    out["raw_val"] = np.concatenate([a.values for a in raw["A"]])
    out["raw_norm"] = np.array([a.norm for a in raw["A"]])
    out["final_len"] = np.array([a.support for a in final])
    out["final_idx"] = np.concatenate([a.indices for a in final])
    out["final_val"] = np.concatenate([a.values for a in final])
    out["final_norm"] = np.array([a.norm for a in final])
    top_k = C1["top_k"]
    for rerank in (True, False):
        tag = "rr" if rerank else "nr"
        rid, rsc = [], []
        for q in qs:
            res, _t = rix.query(bundle, as_viewset("query", q), top_k=top_k, rerank=rerank)
            rid.append([ids.index(r[0]) for r in res])
            rsc.append([r[1] for r in res])
        out[f"q_{tag}_ids"] = np.array(rid, dtype=np.int64)
        out[f"q_{tag}_scores"] = np.array(rsc)
        bid, bsc = [], []
        for i in range(0, len(ids), 125):
            res, _t = rix.query_by_id(bundle, ids[i], top_k=top_k, rerank=rerank)
            bid.append([ids.index(r[0]) for r in res])
            bsc.append([r[1] for r in res])
        out[f"id_{tag}_ids"] = np.array(bid, dtype=np.int64)
        out[f"id_{tag}_scores"] = np.array(bsc)
    out["q_fif_scores"] = np.stack([rmt.query_fif(bundle.fifs["A"], q, ma=C1["ma"]) for q in qs])
    out["q_rerank_scores"] = np.stack([rix.rerank_scores(bundle, {"A": s, "B": s})
                                       for s in out["q_fif_scores"]])
    out["fif_len"] = np.array([len(o) for o in bundle.fifs["A"].entry_ordinals])
    out["fif_ord"] = np.concatenate(bundle.fifs["A"].entry_ordinals)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)
    print("c1 done")


def golden_bundles():
    """The reference's own `save_bundle` directory (index.py:360-375) for the
    tiny and small end-to-end cases, every file's bytes kept verbatim: the
    GPU-built bundle must save to the same bytes (config, shapes, codebooks,
    F-IF lists) and the GPU path must load and serve the reference's files."""
    for case in E2E_CASES[:2]:
        (name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv) = case
        views, _ = mixture_views(seed, N, V, d, classes, zero_views=zv, n_queries=nq)
        db = views[:N]
        ids = shape_ids(N)
        C = sampled_codebook(db, K, seed + 1)
        cfg = rix.IndexConfig(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2, imported=True)
        bundle = reference_bundle(db, ids, C, cfg)[0]
        out = {}
        with tempfile.TemporaryDirectory() as td:
            rix.save_bundle(bundle, td)
            for fn in sorted(os.listdir(td)):
                with open(os.path.join(td, fn), "rb") as fh:
                    out["file:" + fn] = np.frombuffer(fh.read(), dtype=np.uint8)
        np.savez_compressed(os.path.join(HERE, f"bundle_{name}.npz"), **out)
        print("bundle", name, "done")


def golden_exact():
    """Reference rankings with exact=True (index.py:230-243: exact set
    similarity against every database shape), with and without re-ranking."""
    for case in E2E_CASES[:2]:
        (name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv) = case
        views, _ = mixture_views(seed, N, V, d, classes, zero_views=zv, n_queries=nq)
        db, qs = views[:N], views[N:]
        ids = shape_ids(N)
        C = sampled_codebook(db, K, seed + 1)
        cfg = rix.IndexConfig(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2, imported=True)
        bundle = reference_bundle(db, ids, C, cfg)[0]
        out = {}
        for rerank, tag in ((True, "rr"), (False, "nr")):
            rid, rsc = [], []
            for q in qs:
                res, _t = rix.query(bundle, as_viewset("query", q), top_k=top_k, exact=True,
                                    rerank=rerank)
                rid.append([ids.index(r[0]) for r in res])
                rsc.append([r[1] for r in res])
            out[f"x_{tag}_ids"] = np.array(rid, dtype=np.int64)
            out[f"x_{tag}_scores"] = np.array(rsc)
        np.savez_compressed(os.path.join(HERE, f"exact_{name}.npz"), **out)
        print("exact", name, "done")


def golden_eval():
    """Reference evaluate_index (index.py:317-333) with the mixture classes as
    labels: metrics with / without re-ranking, and exact."""
    import dataclasses

    for case in EVAL_CASES:
        (name, seed, N, V, d, classes, K, ma, k1, k2, sigma) = case
        views, labels = mixture_views(seed, N, V, d, classes, sigma=sigma, zero_views=3)
        db = views[:N]
        ids = shape_ids(N)
        C = sampled_codebook(db, K, seed + 1)
        cfg = rix.IndexConfig(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2, imported=True)
        bundle = reference_bundle(db, ids, C, cfg)[0]
        bundle = dataclasses.replace(bundle, labels={ids[i]: f"c{labels[i]}" for i in range(N)})
        out = {}
        for tag, kw in (("rr", dict(rerank=True)), ("nr", dict(rerank=False)),
                        ("x", dict(exact=True, rerank=False))):
            rep = rix.evaluate_index(bundle, **kw)
            out[f"{tag}_metrics"] = np.array([rep.nn, rep.ft, rep.st, rep.map, rep.auc])
            out[f"{tag}_pr11"] = rep.pr11
            out[f"{tag}_counts"] = np.array([rep.n_queries, rep.n_skipped])
        np.savez_compressed(os.path.join(HERE, f"eval_{name}.npz"), **out)
        print("eval", name, "done")


def golden_exact_sets():
    """Reference exact_hausdorff_distance (both variants) and exact_similarity
    (matching.py:39-61) on seeded view-set pairs: unit non-negative rows,
    signed rows (negative cosines), unequal set sizes, identical sets; and
    exact_baseline_report (index.py:336-357) on the evaluation corpora."""
    import dataclasses

    rng = np.random.default_rng(606)
    out = {}
    pairs = []
    for i in range(24):
        d = int(rng.choice([3, 16, 64, 257]))
        vq, vp = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        if i % 3 == 0:
            q, p = unit_nonneg_rows(rng, vq, d), unit_nonneg_rows(rng, vp, d)
        elif i % 3 == 1:
            q = rng.standard_normal((vq, d))
            p = rng.standard_normal((vp, d))
            q /= np.linalg.norm(q, axis=1, keepdims=True)
            p /= np.linalg.norm(p, axis=1, keepdims=True)
        else:
            q = unit_nonneg_rows(rng, vq, d)
            p = q.copy()
        pairs.append((q, p))
    for i, (q, p) in enumerate(pairs):
        out[f"p{i}_q"], out[f"p{i}_p"] = q, p
        out[f"p{i}_out"] = np.array([rmt.exact_hausdorff_distance(q, p, "robust"),
                                     rmt.exact_hausdorff_distance(q, p, "standard"),
                                     rmt.exact_similarity(q, p)])
    out["n_pairs"] = np.array(len(pairs))
    for case in EVAL_CASES:
        (name, seed, N, V, d, classes, K, ma, k1, k2, sigma) = case
        views, labels = mixture_views(seed, N, V, d, classes, sigma=sigma, zero_views=3)
        db = views[:N]
        ids = shape_ids(N)
        C = sampled_codebook(db, K, seed + 1)
        cfg = rix.IndexConfig(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2, imported=True)
        bundle = reference_bundle(db, ids, C, cfg)[0]
        bundle = dataclasses.replace(bundle, labels={ids[i]: f"c{labels[i]}" for i in range(N)})
        rep = rix.exact_baseline_report(bundle, channel="B")
        out[f"{name}_metrics"] = np.array([rep.nn, rep.ft, rep.st, rep.map, rep.auc])
        out[f"{name}_pr11"] = rep.pr11
        out[f"{name}_counts"] = np.array([rep.n_queries, rep.n_skipped])
    np.savez_compressed(os.path.join(HERE, "exact_sets.npz"), **out)
    print("exact sets done")


def golden_kmeans():
    """Reference train_codebook (codebook.py:64-108: k-means++ seeding, Lloyd
    iterations, empty-cluster repair) on the seeded sets of cases.py."""
    out = {}
    for name in KMEANS_CASES:
        x, k, seed, iters = kmeans_inputs(name)
        cb = rcb.train_codebook(x, k, seed=seed, max_iters=iters, channel="A")
        out[f"{name}_centroids"] = cb.centroids
    np.savez_compressed(os.path.join(HERE, "kmeans.npz"), **out)
    print("kmeans done")


def golden_trained_bundle():
    """Reference build_index (index.py:146-227) from two GIFTFT1 feature files
    with no codebooks given: k-means codebooks per channel (index.py:186-193),
    then the F-IF, self-join, re-rank and S-IF.  Saved: the feature files,
    the manifest rows and every file of the reference's saved bundle."""
    x, labels = mixture_views(51, 60, 6, 32, 5, sigma=0.5, zero_views=4)
    rng = np.random.default_rng(52)
    xb = np.abs(x + 0.05 * rng.standard_normal(x.shape)).astype(np.float32)
    ids = shape_ids(60)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        paths = {}
        for ch, feats in (("A", x), ("B", xb)):
            paths[ch] = os.path.join(td, f"feat_{ch}.bin")
            rft.write_features(paths[ch], [as_viewset(s, feats[i], channels=(ch,))
                                           for i, s in enumerate(ids)], ch)
            out[f"feat_{ch}"] = np.frombuffer(open(paths[ch], "rb").read(), dtype=np.uint8)
        rows = [(f"/meshes/{s}.off", f"c{labels[i]}") for i, s in enumerate(ids)]
        cfg = rix.IndexConfig(n_views=6, codebook_size=8, ma=2, k1=5, k2=2)
        bundle = rix.build_index(rows, cfg, feature_files=paths)
        bd = os.path.join(td, "bundle")
        rix.save_bundle(bundle, bd)
        for fn in sorted(os.listdir(bd)):
            out["file:" + fn] = np.frombuffer(open(os.path.join(bd, fn), "rb").read(),
                                              dtype=np.uint8)
    out["labels"] = np.array([f"c{l}" for l in labels])
    np.savez_compressed(os.path.join(HERE, "bundle_trained.npz"), **out)
    print("trained bundle done")


def golden_ingest():
    """A GIFTFT1 file written by the reference's write_features (features.py
    :121-137) from seeded raw rows -- scales 1e-3..1e3, all-zero rows, a
    repeated id, a UTF-8 id -- and the reference's import_features result
    (features.py:140-185: f64 row norm, divide, round to f32)."""
    rng = np.random.default_rng(77)
    ids = ["a", "shape_\u03b2", "c" * 40, "a", "z", "s0009"]
    V, d = 6, 300
    vss = []
    for sid in ids:
        m = rng.standard_normal((V, d)) * 10.0 ** rng.uniform(-3, 3, (V, 1))
        m = np.abs(m).astype(np.float32) if sid != "z" else m.astype(np.float32)
        m[rng.random(V) < 0.25] = 0.0
        vss.append(as_viewset(sid, m, channels=("A",)))
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "feat.bin")
        rft.write_features(path, vss, "A")
        blob = open(path, "rb").read()
        imp = rft.import_features(path, "A")
    out = {"blob": np.frombuffer(blob, dtype=np.uint8),
           "ids": np.array(list(imp), dtype=object).astype(str),
           "mats": np.stack([imp[s].matrix("A") for s in imp])}
    np.savez_compressed(os.path.join(HERE, "ingest.npz"), **out)
    print("ingest done")


if __name__ == "__main__":
    if sys.argv[1:] == ["exact_sets"]:
        golden_exact_sets()
        sys.exit(0)
    if sys.argv[1:] == ["c1"]:
        golden_c1()
        sys.exit(0)
    if sys.argv[1:] == ["ingest"]:
        golden_ingest()
        sys.exit(0)
    if sys.argv[1:] == ["kmeans"]:
        golden_kmeans()
        sys.exit(0)
    if sys.argv[1:] == ["trained"]:
        golden_trained_bundle()
        sys.exit(0)
    if sys.argv[1:] == ["eval"]:
        golden_eval()
        sys.exit(0)
    if sys.argv[1:] == ["bundles"]:
        golden_bundles()
        sys.exit(0)
    if sys.argv[1:] == ["exact"]:
        golden_exact()
        sys.exit(0)
    golden_quantize()
    print("quantize done")
    golden_fif()
    print("fif done")
    golden_rerank()
    print("rerank done")
    golden_e2e()
    golden_bundles()
    golden_exact()
    golden_eval()
    golden_ingest()
    golden_kmeans()
    golden_trained_bundle()
    golden_c1()
    golden_exact_sets()
