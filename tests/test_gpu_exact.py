"""GPU: exact set matching (matching.py:39-61) and the exact-Hausdorff
baseline report (index.py:336-357) against goldens the reference produced
(tests/golden/make_golden.py exact_sets)."""

import numpy as np
import pytest
import torch

from cases import EVAL_CASES, mixture_views, sampled_codebook, shape_ids
from conftest import load_golden

pytestmark = pytest.mark.gpu

import paper_1604_01879_b200 as gift  # noqa: E402
from paper_1604_01879_b200 import matching as mt  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402
from paper_1604_01879_b200.errors import DimensionMismatch, EmptySet  # noqa: E402


def test_exact_functions_against_reference():
    g = load_golden("exact_sets.npz")
    for i in range(int(g["n_pairs"])):
        q, p, ref = g[f"p{i}_q"], g[f"p{i}_p"], g[f"p{i}_out"]
        got = [mt.exact_hausdorff_distance(q, p, "robust"),
               mt.exact_hausdorff_distance(q, p, "standard"), mt.exact_similarity(q, p)]
        # f64 dots in another summation order than the reference's BLAS
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-14, err_msg=f"pair {i}")
        assert mt.exact_hausdorff_distance(q, p) == got[0]  # default variant: robust


def test_exact_functions_errors_and_batch():
    rng = np.random.default_rng(3)
    v = rng.random((4, 6))
    with pytest.raises(EmptySet):
        mt.exact_similarity(np.zeros((0, 6)), v)
    with pytest.raises(DimensionMismatch):
        mt.exact_similarity(v, rng.random((4, 5)))
    with pytest.raises(ValueError):
        mt.exact_hausdorff_distance(v, v, "mean")
    Q = rng.standard_normal((5, 7, 33)).astype(np.float32)
    P = rng.standard_normal((9, 4, 33)).astype(np.float32)
    qc = np.array([7, 3, 1, 7, 5], dtype=np.int32)
    pc = np.array([4, 4, 2, 1, 3, 4, 4, 2, 1], dtype=np.int32)
    out = mt.exact_set_scores(Q, P, qc, pc).cpu().numpy()
    for b in range(5):
        for n in range(9):
            q, p = Q[b, :qc[b]], P[n, :pc[n]]
            exp = [mt.exact_hausdorff_distance(q, p, "robust"),
                   mt.exact_hausdorff_distance(q, p, "standard"), mt.exact_similarity(q, p)]
            np.testing.assert_allclose(out[b, n], exp, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("case", EVAL_CASES, ids=[c[0] for c in EVAL_CASES])
def test_exact_baseline_report_against_reference(case):
    name, seed, N, V, d, classes, K, ma, k1, k2, sigma = case
    g = load_golden("exact_sets.npz")
    views, labels = mixture_views(seed, N, V, d, classes, sigma=sigma, zero_views=3)
    ids = shape_ids(N)
    C = sampled_codebook(views, K, seed + 1)
    cfg = gift.IndexConfig(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2, imported=True)
    bundle = gift.build_index_from_views(
        views, ids, cfg, codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")},
        labels={ids[i]: f"c{labels[i]}" for i in range(N)})
    rep = gift.exact_baseline_report(bundle, channel="B")
    assert [rep.n_queries, rep.n_skipped] == list(g[f"{name}_counts"])
    got = np.array([rep.nn, rep.ft, rep.st, rep.map, rep.auc])
    # identical rankings give identical metrics; a swap of scores tied within
    # the tensor-core scan's 1e-5 tolerance moves a metric by at most ~1 / N
    np.testing.assert_allclose(got, g[f"{name}_metrics"], atol=2.0 / N)
    np.testing.assert_allclose(rep.pr11, g[f"{name}_pr11"], atol=2.0 / N)


def test_eval_ranks_kernel_matches_lexsort():
    """gift_eval_ranks: 1-based ranks of the relevant shapes in a (score
    desc, id rank asc) ordering without the query itself, with ties."""
    from paper_1604_01879_b200 import _native as nat

    rng = np.random.default_rng(9)
    B, N = 6, 3000
    S = np.round(rng.random((B, N)), 2)  # many exact ties
    S[:, ::7] = 0.0
    idrank = rng.permutation(N).astype(np.int32)
    selfs = rng.integers(0, N, B).astype(np.int32)
    R = 300
    rel = np.stack([rng.choice(N, R, replace=False) for _ in range(B)]).astype(np.int32)
    rel[rel == selfs[:, None]] = -1
    rel[2, 150:] = -1
    dev = torch.device("cuda", 0)
    out = torch.empty((B, R), dtype=torch.int32, device=dev)
    sd, ird = torch.from_numpy(S).to(dev), torch.from_numpy(idrank).to(dev)
    sl, rd = torch.from_numpy(selfs).to(dev), torch.from_numpy(rel).to(dev)
    nat.call("gift_eval_ranks", nat.ptr(sd), B, N, nat.ptr(ird), nat.ptr(sl), nat.ptr(rd), R,
             nat.ptr(out), nat.stream_ptr())
    got = out.cpu().numpy()
    for b in range(B):
        keep = np.arange(N) != selfs[b]
        order = np.flatnonzero(keep)[np.lexsort((idrank[keep], -S[b, keep]))]
        pos = np.empty(N, dtype=np.int64)
        pos[order] = np.arange(1, len(order) + 1)
        for r in range(R):
            assert got[b, r] == (pos[rel[b, r]] if rel[b, r] >= 0 else -1)
