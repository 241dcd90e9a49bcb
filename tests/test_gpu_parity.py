"""GPU parity: the CUDA path (through libgift.so) against the reference's
golden vectors and the CPU oracle on the same seeded inputs."""

import io
import os
import tempfile
import types

import numpy as np
import pytest
import torch

import oracle
from cases import E2E_CASES, EVAL_CASES, mixture_views, sampled_codebook, shape_ids, unit_nonneg_rows
from conftest import load_golden
from helpers import RTOL, assert_act_close, assert_ranking_close, unpack_acts, unpack_lists

pytestmark = pytest.mark.gpu

import paper_1604_01879_b200 as gift  # noqa: E402
from paper_1604_01879_b200 import _native as nat  # noqa: E402
from paper_1604_01879_b200 import engine as eg  # noqa: E402
from paper_1604_01879_b200 import matching as mt  # noqa: E402
from paper_1604_01879_b200 import rerank as rr  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook, quantize, quantize_batch  # noqa: E402
from paper_1604_01879_b200.errors import DimensionMismatch, EmptySet  # noqa: E402
from paper_1604_01879_b200.features import ViewSet  # noqa: E402


def dev():
    return torch.device("cuda", 0)


# ---------------------------------------------------------------- K1 quantize
def test_quantize_bit_exact_golden():
    g = load_golden("quantize.npz")
    for i in range(int(g["n_cases"])):
        C, X, ma, out = g[f"c{i}_C"], g[f"c{i}_X"], int(g[f"c{i}_ma"]), g[f"c{i}_out"]
        cb = Codebook(C)
        got = quantize_batch(cb, X, ma)  # f64 inputs
        np.testing.assert_array_equal(got, out, err_msg=f"case {i}")
        if np.array_equal(X.astype(np.float32).astype(np.float64), X):
            np.testing.assert_array_equal(quantize_batch(cb, X.astype(np.float32), ma), out)
        np.testing.assert_array_equal(quantize(cb, X[0], ma), out[0])


@pytest.mark.parametrize("K,d,ma", [(256, 4096, 2), (1024, 4096, 2), (64, 256, 1), (4096, 1024, 1)])
def test_quantize_bit_exact_vs_oracle_config_shapes(K, d, ma):
    views, _ = mixture_views(K + d, max(300, K // 4), 8, d, 20, mu0=-0.26)
    C = sampled_codebook(views, K, 1)
    X = mixture_views(K + d + 1, 120, 8, d, 20, mu0=-0.26)[0].reshape(-1, d)
    got = quantize_batch(Codebook(C), X, ma)
    np.testing.assert_array_equal(got, oracle.quantize_many(C, X, ma))


def test_quantize_fp16_rows_and_ties():
    rng = np.random.default_rng(3)
    C = unit_nonneg_rows(rng, 32, 1024).astype(np.float16).astype(np.float32)
    C[5] = C[17]  # exact duplicate: lower index wins
    X = np.concatenate([C[:8], unit_nonneg_rows(rng, 200, 1024)]).astype(np.float16)
    got = quantize_batch(Codebook(C), torch.from_numpy(X), 3)
    np.testing.assert_array_equal(got, oracle.quantize_many(C, X.astype(np.float64), 3))


def test_quantize_errors():
    cb = Codebook(np.eye(4, dtype=np.float32))
    with pytest.raises(DimensionMismatch):
        quantize(cb, np.zeros(5))
    with pytest.raises(ValueError):
        quantize(cb, np.zeros(4), ma=5)


# ---------------------------------------------------------------- K2 build
def _viewsets(db, ids, channels=("A", "B")):
    return [ViewSet.from_matrix(s, m, channels) for s, m in zip(ids, db)]


@pytest.mark.parametrize("tag", ["k5", "k1"])
def test_build_fif_bit_exact_golden(tag):
    g = load_golden("fif.npz")
    db = g["db"]
    ids = shape_ids(len(db))
    fif = mt.build_fif(_viewsets(db, ids, ("A",)), Codebook(g[f"{tag}_C"], "A"), "A")
    np.testing.assert_array_equal([len(o) for o in fif.entry_ordinals], g[f"{tag}_entry_len"])
    np.testing.assert_array_equal(np.concatenate(fif.entry_ordinals), g[f"{tag}_entry_ord"])
    np.testing.assert_array_equal(np.concatenate(fif.entry_features), g[f"{tag}_entry_feat"])
    np.testing.assert_array_equal(fif.shape_matrix(0), g[f"{tag}_shape_matrix_0"])
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "fif.bin")
        mt.save_fif(fif, p)
        assert open(p, "rb").read() == g[f"{tag}_fif_bytes"].tobytes()
        loaded = mt.load_fif(p, Codebook(g[f"{tag}_C"], "A"))
        q = g["queries"][0]
        np.testing.assert_array_equal(mt.query_fif(loaded, q, 2 if tag == "k5" else 1),
                                      mt.query_fif(fif, q, 2 if tag == "k5" else 1))
    # K3 scores against the reference
    K = len(g[f"{tag}_entry_len"])
    queries = list(g["queries"]) + list(db[:3])
    for ma in sorted({1, min(2, K), K}):
        got = np.stack([mt.query_fif(fif, q, ma) for q in queries])
        np.testing.assert_allclose(got, g[f"{tag}_scores_ma{ma}"], rtol=RTOL, atol=1e-7)
        ref = g[f"{tag}_scores_ma{ma}"]
        assert ((got == 0) == (ref == 0)).all()  # unvisited shapes score exactly 0


def test_build_fif_large_bit_exact_vs_oracle():
    """C2-shaped cells (d=4096, K=256) on 400 shapes: lists bit-exact."""
    views, _ = mixture_views(99, 400, 16, 4096, 55, mu0=-0.26)
    C = sampled_codebook(views, 256, 2)
    assign = oracle.quantize_many(C, views.reshape(-1, 4096), 1).reshape(400, 16)
    ref = oracle.build_fif(list(views), C, assign=assign)
    fif = mt.build_fif_from_tensor(torch.from_numpy(views).to(dev()), Codebook(C), shape_ids(400))
    for a, b in zip(fif.entry_ordinals, ref.entry_ordinals):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(np.concatenate(fif.entry_features),
                                  np.concatenate(ref.entry_features))


# ---------------------------------------------------------------- K3 score
@pytest.mark.parametrize("similarity", ["cosine", "gaussian"])
@pytest.mark.parametrize("ma", [1, 2])
def test_query_fif_vs_oracle_c1_shapes(similarity, ma):
    """Config-1 shapes (d=256, K=64) at N=300: scores within 1e-5 rel."""
    views, _ = mixture_views(7, 300, 64, 256, 40, n_queries=6)
    db, qs = views[:300], views[300:]
    C = sampled_codebook(db, 64, 3)
    assign = oracle.quantize_many(C, db.reshape(-1, 256), 1).reshape(300, 64)
    ref = oracle.build_fif(list(db), C, assign=assign)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev()), Codebook(C), shape_ids(300))
    got = mt.query_fif_batch(fif, qs, ma, similarity).cpu().numpy()
    for q, g in zip(qs, got):
        cells = oracle.quantize_many(C, q.astype(np.float64), ma)
        e = oracle.query_fif(ref, q, ma, similarity, cells=cells)
        np.testing.assert_allclose(g, e, rtol=RTOL, atol=1e-9)
        assert ((g == 0) == (e == 0)).all()


def test_query_fif_degeneracy_and_bounds():
    """K=1 and ma=K equal the exact mean-of-max similarity; scores
    lower-bound it and grow with ma (test_matching.py:127-162)."""
    rng = np.random.default_rng(5)
    mats = np.stack([unit_nonneg_rows(rng, 6, 24) for _ in range(12)])
    exact = np.array([[np.clip(q.astype(np.float64) @ p.astype(np.float64).T, 0, 1).max(1).mean()
                       for p in mats] for q in mats])
    C = sampled_codebook(mats, 5, 0)
    for K in (1, 5):
        fif = mt.build_fif_from_tensor(torch.from_numpy(mats).to(dev()), Codebook(C[:K]),
                                       shape_ids(12))
        prev = None
        for ma in range(1, K + 1):
            s = mt.query_fif_batch(fif, mats, ma).cpu().numpy()
            assert (s <= exact + 1e-6).all()
            if prev is not None:
                assert (s >= prev - 1e-7).all()
            prev = s
        np.testing.assert_allclose(prev, exact, rtol=RTOL, atol=1e-7)
        assert (prev.argmax(axis=1) == np.arange(12)).all()  # self-retrieval


@pytest.mark.parametrize("tag", ["k5", "k1"])
def test_query_fif_f64_matches_reference_goldens(tag):
    """precision="f64" (gift_fif_score_f64): the reference's own query_fif
    scores to f64 rounding (1e-12 absolute, the reference's criterion-3
    tolerance), at every ma including the ma = K degeneracy."""
    g = load_golden("fif.npz")
    db = g["db"]
    ids = shape_ids(len(db))
    fif = mt.build_fif(_viewsets(db, ids, ("A",)), Codebook(g[f"{tag}_C"], "A"), "A")
    K = len(g[f"{tag}_entry_len"])
    queries = list(g["queries"]) + list(db[:3])
    for ma in sorted({1, min(2, K), K}):
        got = np.stack([mt.query_fif(fif, q, ma, precision="f64") for q in queries])
        np.testing.assert_allclose(got, g[f"{tag}_scores_ma{ma}"], rtol=0, atol=1e-12)
        assert ((got == 0) == (g[f"{tag}_scores_ma{ma}"] == 0)).all()


@pytest.mark.parametrize("similarity", ["cosine", "gaussian"])
def test_query_fif_f64_vs_oracle(similarity):
    """The f64 path against the oracle's f64 loops (zero query views, ma = 2,
    config-1 dims): 1e-12 relative."""
    views, _ = mixture_views(17, 120, 16, 256, 12, n_queries=4)
    db, qs = views[:120], views[120:].copy()
    qs[1, 3] = 0.0
    C = sampled_codebook(db, 16, 3)
    assign = oracle.quantize_many(C, db.reshape(-1, 256), 1).reshape(120, 16)
    ref = oracle.build_fif(list(db), C, assign=assign)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev()), Codebook(C), shape_ids(120))
    got = mt.query_fif_batch(fif, qs, 2, similarity, precision="f64").cpu().numpy()
    for q, gq in zip(qs, got):
        cells = oracle.quantize_many(C, q.astype(np.float64), 2)
        e = oracle.query_fif(ref, q, 2, similarity, cells=cells)
        np.testing.assert_allclose(gq, e, rtol=1e-12, atol=1e-15)
        assert ((gq == 0) == (e == 0)).all()
    with pytest.raises(ValueError):
        mt.query_fif_batch(fif, qs, 2, similarity, precision="bf16")
    # queries in workspace-bounded chunks (one query per chunk here): the same
    old_ws = mt.F64_WS_BYTES
    try:
        mt.F64_WS_BYTES = 1
        chunked = mt.query_fif_batch(fif, qs, 2, similarity, precision="f64").cpu().numpy()
    finally:
        mt.F64_WS_BYTES = old_ws
    np.testing.assert_array_equal(chunked, got)


def test_query_fif_f64_degeneracy_is_exact():
    """K = 1 and ma = K: the f64 path equals the exact set similarity to
    1e-12 (the reference's acceptance criterion 1 asks 1e-9)."""
    rng = np.random.default_rng(5)
    mats = np.stack([unit_nonneg_rows(rng, 6, 24) for _ in range(12)])
    exact = np.array([[np.clip(q.astype(np.float64) @ p.astype(np.float64).T, 0, 1).max(1).mean()
                       for p in mats] for q in mats])
    C = sampled_codebook(mats, 5, 0)
    for K in (1, 5):
        fif = mt.build_fif_from_tensor(torch.from_numpy(mats).to(dev()), Codebook(C[:K]),
                                       shape_ids(12))
        s = mt.query_fif_batch(fif, mats, K, precision="f64").cpu().numpy()
        np.testing.assert_allclose(s, exact, rtol=0, atol=1e-12)


def test_zero_views_skipped_and_counted():
    rng = np.random.default_rng(8)
    mats = np.stack([unit_nonneg_rows(rng, 4, 16) for _ in range(5)])
    mats[0, 1] = 0.0
    C = sampled_codebook(mats, 3, 0)
    fif = mt.build_fif_from_tensor(torch.from_numpy(mats).to(dev()), Codebook(C), shape_ids(5))
    assert fif.total_postings == 5 * 4 - 1
    q = mats[2].copy()
    q[0] = 0.0
    ref = oracle.build_fif(list(mats), C)
    np.testing.assert_allclose(mt.query_fif(fif, q, 2), oracle.query_fif(ref, q, 2),
                               rtol=RTOL, atol=1e-9)
    with pytest.raises(EmptySet):
        mt.query_fif(fif, np.zeros((0, 16)), 2)


# ---------------------------------------------------------------- K4/K5/K6
def test_rerank_kernels_golden():
    g = load_golden("rerank.npz")
    S = g["scores"]
    for k in (1, 4, 10, 40):
        for s, ref in zip(S, unpack_acts(g, f"act_k{k}")):
            a = rr.build_activation(s, k)
            np.testing.assert_array_equal(a.indices, ref[0])
            np.testing.assert_array_equal(a.values, ref[1])
            assert a.norm == ref[2]
        for s, ref in zip(S, unpack_lists(g, f"nbr_k{k}", f"nbr_k{k}_len")):
            assert rr.top_neighbors(s, k) == list(ref)
    mk = lambda t: [rr.SparseActivation("x", i, v, n) for i, v, n in t]  # noqa: E731
    a1, a2 = mk(unpack_acts(g, "a1")), mk(unpack_acts(g, "a2"))
    n1 = [list(map(int, x)) for x in unpack_lists(g, "n1", "n1_len")]
    n2 = [list(map(int, x)) for x in unpack_lists(g, "n2", "n2_len")]
    c1, c2 = rr.co_augment(a1, a2, n1, n2)
    for got, ref in zip(c1, unpack_acts(g, "co1")):  # same f64 op order: bit-exact
        np.testing.assert_array_equal(got.indices, ref[0])
        np.testing.assert_array_equal(got.values, ref[1])
        assert got.norm == ref[2]
    for got, ref in zip(c2, unpack_acts(g, "co2")):
        np.testing.assert_array_equal(got.values, ref[1])
    for alpha in (0.25, 0.5, 1.0, 2.0):
        for x, y, ref in zip(c1, c2, unpack_acts(g, f"agg{alpha}")):
            got = rr.aggregate(x, y, alpha)
            np.testing.assert_array_equal(got.indices, ref[0])
            np.testing.assert_allclose(got.values, ref[1], rtol=1e-13, atol=0)
        for x in c1:  # idempotence is exact (rerank.py:142-146)
            got = rr.aggregate(x, x, alpha)
            np.testing.assert_array_equal(got.values, x.values)
    sif = rr.build_sif(c1)
    np.testing.assert_array_equal([len(o) for o in sif.entry_ordinals], g["sif_len"])
    np.testing.assert_array_equal(np.concatenate(sif.entry_ordinals), g["sif_ord"])
    np.testing.assert_array_equal(np.concatenate(sif.entry_values), g["sif_val"])
    np.testing.assert_array_equal(sif.norms, g["sif_norms"])
    got = np.stack([rr.query_sif(sif, q) for q in c1 + c2])
    np.testing.assert_array_equal(got, g["sif_scores"])
    for j, q in enumerate(c1):
        if q.support:
            assert rr.query_sif(sif, q)[j] == 1.0  # self-score exactly 1


def test_rerank_kats():
    a = rr.build_activation([1.0, 0.8, 0.3, 0.1], 2)
    assert dict(a.items()) == {0: 1.0, 1: 0.8}
    assert rr.build_activation([0.0, 0.0, 0.0], 2).support == 0
    assert dict(rr.build_activation([1.0, 0.5, 0.5, 0.2], 2).items()) == {0: 1.0, 1: 0.5}
    assert rr.top_neighbors([0.2, 1.0, 0.5, 0.5], 3) == [1, 2, 3]
    assert rr.top_neighbors([0.0, 0.0], 2) == []
    f = rr.aggregate(rr.make_activation("a", [0], [0.25]), rr.make_activation("a", [0], [0.81]), 0.5)
    assert abs(f.values[0] - 0.49) <= 1e-12
    with pytest.raises(ValueError):
        rr.build_sif([rr.make_activation("a", [3], [0.5])])


def test_topk_large_rows_vs_lexsort():
    rng = np.random.default_rng(11)
    S = np.round(rng.random((7, 50_000)), 3)
    S[:, ::7] = 0.0
    t = torch.from_numpy(S).to(dev())
    for k in (1, 4, 10, 100, 700, 2048):
        idx, val = eg.topk_rows(t, k)
        for r in range(7):
            ref = np.lexsort((np.arange(S.shape[1]), -S[r]))[:k]
            np.testing.assert_array_equal(idx[r].cpu().numpy(), ref)


# ---------------------------------------------------------------- end to end
def _e2e_bundle(case, storage="float32", similarity="cosine"):
    name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv = case
    views, _ = mixture_views(seed, N, V, d, classes, zero_views=zv, n_queries=nq)
    db, qs = views[:N], views[N:]
    ids = shape_ids(N)
    C = sampled_codebook(db, K, seed + 1)
    cfg = gift.IndexConfig(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2, imported=True,
                           storage_dtype=storage, similarity=similarity)
    bundle = gift.build_index_from_views(db, ids, cfg,
                                         codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")})
    return bundle, db, qs, ids, C


@pytest.mark.parametrize("case", E2E_CASES, ids=[c[0] for c in E2E_CASES])
def test_end_to_end_against_reference(case):
    name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv = case
    g = load_golden(f"e2e_{name}.npz")
    bundle, db, qs, ids, C = _e2e_bundle(case)
    # stage-wise: raw activations and final (augmented) activations
    raw = bundle.raw_activations["A"]
    for i, ref in enumerate(unpack_acts(g, "raw")):
        a = raw[i]
        assert_act_close((a.indices, a.values, a.norm), ref)
    # F-IF and re-rank scores of the queries
    sc = mt.query_fif_batch(bundle.fifs["A"], qs, ma).cpu().numpy()
    np.testing.assert_allclose(sc, g["q_fif_scores"], rtol=RTOL, atol=1e-9)
    rs = np.stack([gift.rerank_scores(bundle, {"A": s, "B": s}) for s in g["q_fif_scores"]])
    np.testing.assert_allclose(rs, g["q_rerank_scores"], rtol=RTOL, atol=1e-12)
    for rerank, tag in ((True, "rr"), (False, "nr")):
        batch = gift.query_batch(bundle, qs, top_k=top_k, rerank=rerank)
        for qi, q in enumerate(qs):
            res, tim = gift.query(bundle, ViewSet.from_matrix("query", q), top_k=top_k,
                                  rerank=rerank)
            assert set(tim) == {"render", "match"}
            assert res == batch[qi]
            assert_ranking_close([ids.index(r[0]) for r in res], [r[1] for r in res],
                                 g[f"q_{tag}_ids"][qi], g[f"q_{tag}_scores"][qi])
        for j, i in enumerate(range(0, N, max(1, N // 8))):
            res, _ = gift.query_by_id(bundle, ids[i], top_k=top_k, rerank=rerank)
            assert res[0][0] == ids[i]  # self-retrieval ranks first
            assert_ranking_close([ids.index(r[0]) for r in res], [r[1] for r in res],
                                 g[f"id_{tag}_ids"][j], g[f"id_{tag}_scores"][j])


def test_persistence_round_trip_and_bytes():
    bundle, db, qs, ids, C = _e2e_bundle(E2E_CASES[1])
    with tempfile.TemporaryDirectory() as td:
        d1 = gift.save_bundle(bundle, os.path.join(td, "a"))
        d2 = gift.save_bundle(bundle, os.path.join(td, "b"))
        for f in sorted(os.listdir(d1)):
            assert open(os.path.join(d1, f), "rb").read() == open(os.path.join(d2, f), "rb").read()
        loaded = gift.load_bundle(d1)
        assert loaded.shape_ids == bundle.shape_ids and loaded.config == bundle.config
        for sid in ids[:5]:
            assert gift.query_by_id(loaded, sid, top_k=20)[0] == gift.query_by_id(bundle, sid, top_k=20)[0]


@pytest.mark.parametrize("variant", ["default", "pair", "static"])
def test_fp16_storage_matches_widened_oracle(variant):
    """Config 4 storage (D5): fp16 features, fp32 accumulation; the oracle
    sees the same fp16 values widened to f32.  Variants (view flags): the
    single-CTA scan with two epilogue groups (default), CTA pairs
    (GIFT_FIF_PAIR_ON) and the static item stride (GIFT_FIF_SCHED_STATIC)."""
    views, _ = mixture_views(21, 200, 20, 1024, 16, n_queries=4)
    v16 = views.astype(np.float16)
    db, qs = v16[:200], v16[200:].astype(np.float32)
    C = sampled_codebook(db.astype(np.float32), 32, 1)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev()), Codebook(C), shape_ids(200))
    fif.dev.set_variant(pair="on" if variant == "pair" else "auto",
                        sched="static" if variant == "static" else "dynamic")
    dbw = db.astype(np.float32)
    assign = oracle.quantize_many(C, dbw.reshape(-1, 1024), 1).reshape(200, 20)
    ref = oracle.build_fif(list(dbw), C, assign=assign)
    for a, b in zip(fif.entry_ordinals, ref.entry_ordinals):
        np.testing.assert_array_equal(a, b)
    got = mt.query_fif_batch(fif, qs, 1, "gaussian").cpu().numpy()
    for q, gsc in zip(qs, got):
        e = oracle.query_fif(ref, q, 1, "gaussian", cells=oracle.quantize_many(C, q.astype(np.float64), 1))
        np.testing.assert_allclose(gsc, e, rtol=RTOL, atol=1e-9)


def test_sif_self_score_exactly_one_at_scale():
    """A DB shape's own final activation scores exactly 1.0 against itself
    (test_rerank.py:249-253): sequential f64 accumulation == cached norm."""
    bundle, db, qs, ids, C = _e2e_bundle(E2E_CASES[2])
    cfg = bundle.config
    s = mt.query_fif_batch(bundle.fifs["A"], db[:64], cfg.ma)  # the self-join's scores
    nbr, _ = eg.topk_rows(s, cfg.k2, positive_only=True)
    fa = eg.act_mean(bundle.raw_activations["A"].rows, nbr)
    sc = bundle.sif.dev.query(fa).cpu().numpy()
    cnt = fa.cnt.cpu().numpy()
    assert cnt.min() > 0
    for j in range(64):
        assert sc[j, j] == 1.0


@pytest.mark.parametrize("lanes,reserve,graph", [(1, 0, False), (2, 0, False), (3, 20, False),
                                                 (1, 0, True), (3, 20, True)])
def test_query_many_pipelined_equals_batch(lanes, reserve, graph):
    """Batches in flight on 1-3 compute streams (own scratch each; the scan
    optionally leaving SMs to the other lanes; full batches optionally
    replaying each lane's CUDA graph, the ragged last one eager) return the
    serial results, bit for bit -- twice, so the second call replays the
    graphs the first captured."""
    bundle, db, qs, ids, C = _e2e_bundle(E2E_CASES[2])
    host = torch.from_numpy(np.concatenate([qs, db[:21]])).pin_memory()
    for _ in range(2 if graph else 1):
        idx, val = gift.query_many(bundle, host, top_k=30, batch_size=5, lanes=lanes,
                                   reserve_sms=reserve, graph=graph)
    ref = gift.query_batch(bundle, host.numpy(), top_k=30)
    for r in range(len(ref)):
        assert [ids[i] for i in idx[r]] == [x[0] for x in ref[r]]
        np.testing.assert_array_equal(val[r], [x[1] for x in ref[r]])


@pytest.mark.parametrize("similarity", ["gaussian", "cosine"])
def test_tensor_core_scan_matches_oracle_at_c2_dims(similarity):
    """The tcgen05 scan (default for d % 8 == 0) and the CUDA-core scan both
    match the f64 oracle at config-2 dimensions (d = 4096, K = 256, ma = 2)."""
    views, _ = mixture_views(55, 300, 16, 4096, 55, mu0=-0.26, n_queries=8)
    db, qs = views[:300], views[300:]
    C = sampled_codebook(db, 256, 4)
    assign = oracle.quantize_many(C, db.reshape(-1, 4096), 1).reshape(300, 16)
    ref = oracle.build_fif(list(db), C, assign=assign)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev()), Codebook(C), shape_ids(300))
    assert fif.dev.feat_hi is not None  # tensor-core planes built
    got = {}
    # tc: CTA pairs (default with the f32 lo plane); tc_single: one CTA, two
    # epilogue groups; tc_static: static item stride instead of the counter
    for impl, kw in (("tc", {}), ("tc_single", {"pair": "off"}),
                     ("tc_static", {"sched": "static"}), ("simt", {"scan": "simt"})):
        fif.dev.set_variant(**kw)
        got[impl] = mt.query_fif_batch(fif, qs, 2, similarity).cpu().numpy()
    fif.dev.set_variant()
    np.testing.assert_array_equal(got["tc_static"], got["tc"])  # same items, same order
    worst = 0.0
    for i, q in enumerate(qs):
        e = oracle.query_fif(ref, q, 2, similarity,
                             cells=oracle.quantize_many(C, q.astype(np.float64), 2))
        nz = e > 0
        g_tc = got["tc"][i]
        worst = max(worst, float(np.max(np.abs(g_tc[nz] - e[nz]) / e[nz])) if nz.any() else 0.0)
        for impl in ("tc", "tc_single", "simt"):
            np.testing.assert_allclose(got[impl][i], e, rtol=RTOL, atol=1e-12)
            assert ((got[impl][i] == 0) == (e == 0)).all()
    print(f"max relative error tc vs oracle ({similarity}): {worst:.2e}")


@pytest.mark.parametrize("impl", ["tc", "simt"])
def test_quantize_near_ties_and_scale(impl):
    """Bit-exact assignment under stress: midpoints of centroid pairs (d2 ties
    up to rounding), exact duplicates (ties -> lower index), and 8k config-2
    views, on both stage-1 implementations (tensor cores / CUDA cores)."""
    views, _ = mixture_views(321, 200, 16, 4096, 55, mu0=-0.26)
    C = sampled_codebook(views, 256, 9)
    C[200] = C[17]  # exact duplicate centroids
    rng = np.random.default_rng(4)
    a, b = rng.integers(0, 256, 300), rng.integers(0, 256, 300)
    mids = ((C[a].astype(np.float64) + C[b].astype(np.float64)) / 2).astype(np.float32)
    X = np.concatenate([mids, C[:50], mixture_views(322, 500, 16, 4096, 55, mu0=-0.26)[0]
                        .reshape(-1, 4096)]).astype(np.float32)
    cb = Codebook(C)
    for ma in (1, 2, 3):
        got = eg.quantize_rows(cb.device(), torch.from_numpy(X).to(dev()), ma,
                               flags=nat.QUANT_SIMT if impl == "simt" else 0).cpu().numpy()
        np.testing.assert_array_equal(got, oracle.quantize_many(C, X.astype(np.float64), ma))


@pytest.mark.parametrize("V,ma,K", [(16, 1, 32), (16, 2, 32), (20, 3, 16), (64, 2, 64), (70, 2, 64)])
def test_gather_reduce_equals_range_reduce(V, ma, K):
    """The shape-centric gather and owner reduces (available when the index
    has its shape -> segment map and V * ma <= 128) are bit-identical to the
    per-range reduce: same per-view maxima, same ascending-view f64 sum.  Uniform
    random views spread each shape over many cells (> 4 segments: the
    uncached segment path); V * ma = 140 falls back to the range reduce."""
    rng = np.random.default_rng(V * 100 + ma)
    N, d = 300, 64
    db = unit_nonneg_rows(rng, N * V, d).reshape(N, V, d)
    db[rng.random((N, V)) < 0.05] = 0.0  # empty views
    qs = unit_nonneg_rows(rng, 9 * V, d).reshape(9, V, d)
    qs[0, 3] = 0.0
    C = sampled_codebook(db, K, 5)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev()), Codebook(C), shape_ids(N))
    Q = torch.from_numpy(qs).to(dev())
    run = eg.ScoreRunner()
    got = {}
    for impl in ("gather", "range", "owner"):
        fif.dev.set_variant(reduce=impl)
        for sim in ("cosine", "gaussian"):
            s, cs, ci = run.score(fif.dev, Q, ma, mt.sim_mode(sim), 0.5, cand_k=4)
            nbr, val = eg.topk_candidates(cs, ci, 4, positive_only=True)
            got[impl, sim] = (s.cpu().numpy(), nbr.cpu().numpy(), val.cpu().numpy())
    for sim in ("cosine", "gaussian"):
        for impl in ("gather", "owner"):
            for t in range(3):
                np.testing.assert_array_equal(got[impl, sim][t], got["range", sim][t])
        ref = eg.topk_rows(torch.from_numpy(got["range", sim][0]).to(dev()), 4,
                           positive_only=True)[0].cpu().numpy()
        np.testing.assert_array_equal(got["gather", sim][1], ref)
    # candidates-only mode (no dense scores) gives the same neighbour lists
    for impl in ("gather", "range", "owner"):
        fif.dev.set_variant(reduce=impl)
        s, cs, ci = run.score(fif.dev, Q, ma, mt.sim_mode("cosine"), 0.5, cand_k=4, dense=False)
        assert s is None
        nbr, _ = eg.topk_candidates(cs, ci, 4, positive_only=True)
        np.testing.assert_array_equal(nbr.cpu().numpy(), got["gather", "cosine"][1])


_SIF_FLAGS = {"rows": nat.SIF_ROWS, "sort": nat.SIF_SORT, "bucket": nat.SIF_BUCKET}


@pytest.mark.parametrize("mode", ["rows", "sort", "bucket"])
@pytest.mark.parametrize("k", [1, 10, 100, 256])
def test_sparse_sif_ranking_equals_dense(k, mode):
    """Sparse S-IF query + ranking (touched shapes + zero-score fill) is
    identical to top-k over the dense query_sif rows: shuffled id ranks,
    self inside / outside the touched set, an empty query support (pure
    fill), fewer touched shapes than k; repeated calls (scratch re-zeroed).
    All three implementations: per-query accumulator rows, the sort-based one
    (GIFT_SIF_SORT: (query, shape) pairs radix-sorted, runs summed in order)
    and the bucketed one (GIFT_SIF_BUCKET: pairs split by shape range, reduced
    in shared memory)."""
    flags = _SIF_FLAGS[mode]
    rng = np.random.default_rng(k)
    N, B = 500, 37
    acts = []
    for j in range(N):
        idx = np.sort(rng.choice(N, size=rng.integers(1, 6), replace=False))
        val = rng.random(len(idx)) + 0.01
        acts.append(types.SimpleNamespace(indices=idx, values=val, norm=float(np.sum(val))))
    raw = eg.ActRows.from_host(acts, 5)
    sif = eg.DeviceSif.build(raw, N)
    nbr = torch.from_numpy(rng.integers(-1, N, size=(B, 4)).astype(np.int32)).to(dev())
    nbr[0] = -1  # empty support: zero-score fill only
    q = eg.act_mean(raw, nbr)
    rank = rng.permutation(N).astype(np.int32)
    idrank = torch.from_numpy(rank).to(dev())
    order = torch.from_numpy(np.argsort(rank).astype(np.int32)).to(dev())
    self_local = torch.from_numpy(rng.integers(0, N, size=B).astype(np.int32)).to(dev())
    self_local[1] = nbr[1, 0].clamp(min=0)  # self likely touched
    kk = min(k, N)
    di, dv = eg.topk_rows(sif.query(q), kk, idrank=idrank, self_local=self_local)
    for _ in range(2):
        si, sv = sif.query_topk(q, kk, order, idrank, self_local, flags=flags)
        np.testing.assert_array_equal(si.cpu().numpy(), di.cpu().numpy())
        np.testing.assert_array_equal(sv.cpu().numpy(), dv.cpu().numpy())
    assert all(float(a.abs().sum()) == 0.0 for a in sif._acc.values())


@pytest.mark.parametrize("n_shapes", [2048, 9001, 70000])
def test_bucketed_sif_many_buckets_and_conflicts(n_shapes):
    """Bucketed S-IF query over several shape buckets (2^11 shapes each) with
    long postings (few coordinates -> one shape hit by many entries of a
    query, conflicting lanes inside a 32-pair chunk): rankings and f64
    scores bit-equal to the dense rows and to the other two paths."""
    rng = np.random.default_rng(n_shapes)
    N, B, coords = n_shapes, 45, 400
    acts = []
    for j in range(N):
        idx = np.sort(rng.choice(coords, size=rng.integers(1, 9), replace=False))
        val = rng.random(len(idx)) + 0.01
        acts.append(types.SimpleNamespace(indices=idx, values=val, norm=float(np.sum(val))))
    raw = eg.ActRows.from_host(acts, 8)
    sif = eg.DeviceSif.build(raw, coords)
    nbr = torch.from_numpy(rng.integers(-1, N, size=(B, 6)).astype(np.int32)).to(dev())
    q = eg.act_mean(raw, nbr)
    rank = rng.permutation(N).astype(np.int32)
    idrank = torch.from_numpy(rank).to(dev())
    order = torch.from_numpy(np.argsort(rank).astype(np.int32)).to(dev())
    self_local = torch.from_numpy(rng.integers(0, N, size=B).astype(np.int32)).to(dev())
    k = 100
    di, dv = eg.topk_rows(sif.query(q), k, idrank=idrank, self_local=self_local)
    for mode in ("bucket", "rows", "sort", "bucket"):
        si, sv = sif.query_topk(q, k, order, idrank, self_local, flags=_SIF_FLAGS[mode])
        np.testing.assert_array_equal(si.cpu().numpy(), di.cpu().numpy())
        np.testing.assert_array_equal(sv.cpu().numpy(), dv.cpu().numpy())


@pytest.mark.parametrize("case", E2E_CASES[:2], ids=[c[0] for c in E2E_CASES[:2]])
def test_exact_ranking_against_reference(case):
    """query(exact=True): every view probes every cell (ma = K) = the
    reference's exact set similarity (index.py:230-243); rankings with and
    without re-ranking match the reference's (golden exact_*.npz)."""
    name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv = case
    g = load_golden(f"exact_{name}.npz")
    bundle, db, qs, ids, C = _e2e_bundle(case)
    for rerank, tag in ((True, "rr"), (False, "nr")):
        for qi, q in enumerate(qs):
            res, _ = gift.query(bundle, ViewSet.from_matrix("query", q), top_k=top_k,
                                exact=True, rerank=rerank)
            assert_ranking_close([ids.index(r[0]) for r in res], [r[1] for r in res],
                                 g[f"x_{tag}_ids"][qi], g[f"x_{tag}_scores"][qi])


@pytest.mark.parametrize("case", EVAL_CASES, ids=[c[0] for c in EVAL_CASES])
def test_evaluate_index_against_reference(case):
    """evaluate_index (index.py:317-333; NN/FT/ST/MAP/AUC of evaluation.py)
    with re-ranking, without, and exact, against the reference's reports on
    overlapping classes (golden eval_*.npz)."""
    name, seed, N, V, d, classes, K, ma, k1, k2, sigma = case
    g = load_golden(f"eval_{name}.npz")
    views, labels = mixture_views(seed, N, V, d, classes, sigma=sigma, zero_views=3)
    ids = shape_ids(N)
    C = sampled_codebook(views, K, seed + 1)
    cfg = gift.IndexConfig(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2, imported=True)
    bundle = gift.build_index_from_views(
        views, ids, cfg, codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")},
        labels={ids[i]: f"c{labels[i]}" for i in range(N)})
    for tag, kw in (("rr", dict(rerank=True)), ("nr", dict(rerank=False)),
                    ("x", dict(exact=True, rerank=False))):
        rep = gift.evaluate_index(bundle, **kw)
        got = np.array([rep.nn, rep.ft, rep.st, rep.map, rep.auc])
        assert [rep.n_queries, rep.n_skipped] == list(g[f"{tag}_counts"])
        # identical rankings give identical metrics; a swap of scores tied
        # within the 1e-5 tolerance moves a metric by at most ~1 / N
        np.testing.assert_allclose(got, g[f"{tag}_metrics"], atol=2.0 / N)
        np.testing.assert_allclose(rep.pr11, g[f"{tag}_pr11"], atol=2.0 / N)
