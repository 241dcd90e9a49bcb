"""Pins the CPU oracle (oracle/) to golden vectors produced by the reference
implementation itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle
from cases import E2E_CASES, mixture_views, sampled_codebook, shape_ids
from conftest import load_golden
from helpers import unpack_acts, unpack_lists


def test_quantize_exact_against_reference():
    g = load_golden("quantize.npz")
    for i in range(int(g["n_cases"])):
        C, X, ma, out = g[f"c{i}_C"], g[f"c{i}_X"], int(g[f"c{i}_ma"]), g[f"c{i}_out"]
        got = np.stack([oracle.quantize(C, x, ma) for x in X])
        np.testing.assert_array_equal(got, out)
        np.testing.assert_array_equal(oracle.quantize_many(C, X, ma), out)


def test_quantize_many_c_pairwise_matches_numpy_rows(rng):
    C = rng.random((64, 4096)).astype(np.float32)
    X = rng.random((40, 4096))
    dd = oracle.reference_port.sqdist_exact(C, X)
    for i in range(len(X)):
        diffs = C.astype(np.float64) - X[i]
        np.testing.assert_array_equal(dd[i], (diffs * diffs).sum(axis=1))


@pytest.mark.parametrize("tag", ["k5", "k1"])
def test_build_fif_against_reference(tag):
    g = load_golden("fif.npz")
    fif = oracle.build_fif(list(g["db"]), g[f"{tag}_C"])
    lens = g[f"{tag}_entry_len"]
    np.testing.assert_array_equal([len(o) for o in fif.entry_ordinals], lens)
    np.testing.assert_array_equal(np.concatenate(fif.entry_ordinals), g[f"{tag}_entry_ord"])
    np.testing.assert_array_equal(np.concatenate(fif.entry_features), g[f"{tag}_entry_feat"])
    np.testing.assert_array_equal(fif.shape_matrix(0), g[f"{tag}_shape_matrix_0"])
    K = len(lens)
    queries = list(g["queries"]) + list(g["db"][:3])
    for ma in sorted({1, min(2, K), K}):
        got = np.stack([oracle.query_fif(fif, q, ma) for q in queries])
        np.testing.assert_allclose(got, g[f"{tag}_scores_ma{ma}"], rtol=0, atol=1e-12)


def test_rerank_functions_against_reference():
    g = load_golden("rerank.npz")
    S = g["scores"]
    for k in (1, 4, 10, 40):
        ref = unpack_acts(g, f"act_k{k}")
        for s, (ri, rv, rn) in zip(S, ref):
            a = oracle.build_activation(s, k)
            np.testing.assert_array_equal(a.idx, ri)
            np.testing.assert_array_equal(a.val, rv)
            assert a.norm == rn
        nb = unpack_lists(g, f"nbr_k{k}", f"nbr_k{k}_len")
        for s, r in zip(S, nb):
            assert oracle.top_neighbors(s, k) == list(r)
    a1 = [oracle.Act(i, v, n) for i, v, n in unpack_acts(g, "a1")]
    a2 = [oracle.Act(i, v, n) for i, v, n in unpack_acts(g, "a2")]
    n1 = [list(x) for x in unpack_lists(g, "n1", "n1_len")]
    n2 = [list(x) for x in unpack_lists(g, "n2", "n2_len")]
    c1, c2 = oracle.co_augment(a1, a2, n1, n2)
    for got, ref in zip(c1, unpack_acts(g, "co1")):
        np.testing.assert_array_equal(got.idx, ref[0])
        np.testing.assert_array_equal(got.val, ref[1])
        assert got.norm == ref[2]
    for got, ref in zip(c2, unpack_acts(g, "co2")):
        np.testing.assert_array_equal(got.val, ref[1])
    for alpha in (0.25, 0.5, 1.0, 2.0):
        for x, y, ref in zip(c1, c2, unpack_acts(g, f"agg{alpha}")):
            got = oracle.aggregate(x, y, alpha)
            np.testing.assert_array_equal(got.idx, ref[0])
            np.testing.assert_array_equal(got.val, ref[1])
    sif = oracle.build_sif(c1)
    np.testing.assert_array_equal([len(o) for o in sif.entry_ordinals], g["sif_len"])
    np.testing.assert_array_equal(np.concatenate(sif.entry_ordinals), g["sif_ord"])
    np.testing.assert_array_equal(np.concatenate(sif.entry_values), g["sif_val"])
    np.testing.assert_array_equal(sif.norms, g["sif_norms"])
    got = np.stack([oracle.query_sif(sif, q) for q in c1 + c2])
    np.testing.assert_array_equal(got, g["sif_scores"])


@pytest.mark.parametrize("case", E2E_CASES[:2], ids=[c[0] for c in E2E_CASES[:2]])
def test_pipeline_against_reference(case):
    name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv = case
    g = load_golden(f"e2e_{name}.npz")
    views, _ = mixture_views(seed, N, V, d, classes, zero_views=zv, n_queries=nq)
    db, qs = views[:N], views[N:]
    ids = shape_ids(N)
    C = sampled_codebook(db, K, seed + 1)
    np.testing.assert_array_equal(C, g["C"])
    idx = oracle.OracleIndex(list(db), C, ids, ma=ma, k1=k1, k2=k2)
    if g["db_scores"].size:
        np.testing.assert_allclose(np.stack(idx.db_scores["A"]), g["db_scores"], atol=1e-12)
    for got, ref in zip(idx.raw["A"], unpack_acts(g, "raw")):
        np.testing.assert_array_equal(got.idx, ref[0])
        np.testing.assert_allclose(got.val, ref[1], atol=1e-12)
    for got, ref in zip(idx.final, unpack_acts(g, "final")):
        np.testing.assert_array_equal(got.idx, ref[0])
        np.testing.assert_allclose(got.val, ref[1], atol=1e-12)
    for rerank, tag in ((True, "rr"), (False, "nr")):
        for qi, q in enumerate(qs):
            res, _ = idx.query(q, top_k=top_k, rerank=rerank)
            assert [ids.index(r) for r, _s in res] == list(g[f"q_{tag}_ids"][qi])
            np.testing.assert_allclose([s for _r, s in res], g[f"q_{tag}_scores"][qi], atol=1e-12)
        for j, i in enumerate(range(0, N, max(1, N // 8))):
            res, _ = idx.query_by_id(ids[i], top_k=top_k, rerank=rerank)
            assert [ids.index(r) for r, _s in res] == list(g[f"id_{tag}_ids"][j])


def test_gaussian_restatement_properties(rng):
    """Gaussian mode has no reference (D1): pin its properties instead —
    K=1 and ma=K degenerate to the exact mean-of-max Gaussian similarity,
    scores lower-bound it and grow with ma."""
    mats = [oracle.reference_port.np.asarray(m) for m in
            mixture_views(3, 10, 5, 12, 3)[0]]
    def exact(q, p, sigma=0.5):
        d2 = ((q[:, None, :].astype(np.float64) - p[None].astype(np.float64)) ** 2).sum(-1)
        return np.exp(-d2 / sigma ** 2).max(axis=1).mean()
    C = sampled_codebook(np.stack(mats), 4, 1)
    for K, cb in ((1, C[:1]), (4, C)):
        fif = oracle.build_fif(mats, cb)
        for q in mats[:3]:
            ex = np.array([exact(q, p) for p in mats])
            prev = None
            for ma in range(1, K + 1):
                s = oracle.query_fif(fif, q, ma, similarity="gaussian")
                assert (s <= ex + 1e-12).all()
                if prev is not None:
                    assert (s >= prev - 1e-15).all()
                prev = s
            np.testing.assert_allclose(prev, ex, atol=1e-12)


def test_evaluation_metrics_restatement():
    """paper_1604_01879_b200.evaluation restates evaluation.py:44-88: known
    rankings (host-only)."""
    from paper_1604_01879_b200 import evaluation as ev
    from paper_1604_01879_b200.errors import NoValidQueries, SingletonClass

    m = ev.score_ranking("a", ["a", "b", "a", "b", "b"], 3)  # relevant at ranks 1 and 3
    assert (m.nn, m.ft, m.st) == (1.0, 0.5, 1.0)
    assert m.ap == pytest.approx((1 / 1 + 2 / 3) / 2)
    np.testing.assert_allclose(m.pr11, [1.0] * 6 + [2 / 3] * 5)
    m2 = ev.score_ranking("a", ["b", "b", "b"], 2)
    assert (m2.nn, m2.ft, m2.ap) == (0.0, 0.0, 0.0)
    rep = ev.aggregate_report([m, m2], n_skipped=1)
    assert rep.n_queries == 2 and rep.nn == 0.5
    with pytest.raises(SingletonClass):
        ev.score_ranking("a", ["b"], 1)
    with pytest.raises(NoValidQueries):
        ev.aggregate_report([])
