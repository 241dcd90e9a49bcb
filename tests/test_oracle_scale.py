"""CPU: the config-scale oracle (oracle/scale.py) is the loop restatement
(oracle/reference_port.py, itself pinned to the reference's goldens)
reorganised -- check that it computes the same thing."""

import numpy as np
import pytest

import oracle
from cases import E2E_CASES, mixture_views, sampled_codebook, shape_ids
from conftest import load_golden
from helpers import unpack_acts
from oracle import scale


@pytest.mark.parametrize("similarity", ["cosine", "gaussian"])
@pytest.mark.parametrize("ma", [1, 2, 3])
def test_fif_scores_many_equals_loop_restatement(similarity, ma):
    views, _ = mixture_views(7, 150, 10, 48, 8, zero_views=6, n_queries=7)
    db, qs = views[:150], views[150:]
    qs[2, 4] = 0.0  # a zero query view (skipped, still counted)
    C = sampled_codebook(db, 12, 2)
    idx = scale.OracleCsrIndex.from_views(db, C, ma, 6, 3, similarity, self_join=False)
    got = idx.scores(qs)
    ref = oracle.build_fif(list(db), C)
    for q, g in zip(qs, got):
        np.testing.assert_allclose(g, oracle.query_fif(ref, q, ma, similarity), rtol=1e-12,
                                   atol=1e-15)
    # chunked cells (postings split across GEMM blocks) give the same maxima
    got2 = scale.fif_scores_many(idx.cell_off, idx.post_ord, idx.feat_rows, qs,
                                 scale.quantize_many_mt(C, qs.reshape(-1, 48), ma)
                                 .reshape(7, 10, ma), 150, similarity, cell_chunk=7)
    assert (~qs.any(axis=2)).sum() >= 1  # zero query views present
    np.testing.assert_allclose(got2, got, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("case", E2E_CASES, ids=[c[0] for c in E2E_CASES])
def test_lists_and_self_join_equal_loop_restatement(case):
    name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv = case
    views, _ = mixture_views(seed, N, V, d, classes, zero_views=zv, n_queries=nq)
    db = views[:N]
    C = sampled_codebook(db, K, seed + 1)
    idx = scale.OracleCsrIndex.from_views(db, C, ma, k1, k2, "cosine")
    g = load_golden(f"e2e_{name}.npz")  # the reference's own raw and final activations
    for a, (i, v, n) in zip(idx.raw, unpack_acts(g, "raw")):
        np.testing.assert_array_equal(a.idx, i)
        np.testing.assert_allclose(a.val, v, rtol=1e-12)
    for a, (i, v, n) in zip(idx.final, unpack_acts(g, "final")):
        np.testing.assert_array_equal(a.idx, i)
        np.testing.assert_allclose(a.val, v, rtol=1e-12)
    ref = oracle.OracleIndex(list(db), C, shape_ids(N), ma=ma, k1=k1, k2=k2)
    for a, b in zip(idx.sif.entry_ordinals, ref.sif.entry_ordinals):
        np.testing.assert_array_equal(a, b)


def test_build_context_arrays_equals_dict_loops():
    rng = np.random.default_rng(1)
    N, k1, k2 = 400, 10, 4
    raw, ri, rv, rc = [], np.full((N, k1), -1), np.zeros((N, k1)), np.zeros(N, int)
    for j in range(N):
        n = int(rng.integers(0, k1 + 1))
        idx = np.sort(rng.choice(N, n, replace=False))
        val = rng.random(n) + 1e-3
        raw.append(oracle.make_activation(idx, val))
        ri[j, :n], rv[j, :n], rc[j] = idx, val, n
    nbr = np.full((N, k2), -1)
    for j in range(N):
        m = int(rng.integers(0, k2 + 1))
        nbr[j, :m] = rng.choice(N, m, replace=False)
    nb = [[int(x) for x in row if x >= 0] for row in nbr]
    final, sif = scale.build_context(raw, nb)
    fi, fv, fc, norms, sif2 = scale.build_context_arrays(ri, rv, rc, nbr)
    for j, a in enumerate(final):
        np.testing.assert_array_equal(fi[j, :fc[j]], a.idx)
        np.testing.assert_array_equal(fv[j, :fc[j]], a.val)  # same f64 op order: exact
        assert norms[j] == a.norm
    for a, b, c, e in zip(sif.entry_ordinals, sif2.entry_ordinals, sif.entry_values,
                          sif2.entry_values):
        np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(c, e)


def test_topk_stable_equals_lexsort():
    rng = np.random.default_rng(5)
    S = np.round(rng.random((40, 500)), 2)  # ties
    S[:, ::3] = 0.0
    for k in (1, 4, 10, 77):
        top = scale.topk_stable(S, k)
        for r in range(S.shape[0]):
            np.testing.assert_array_equal(top[r], np.lexsort((np.arange(500), -S[r]))[:k])
