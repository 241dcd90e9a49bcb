"""GPU edge cases of the query path against the oracle: a one-shape index,
all-zero queries (pure zero-score fill), top_k above N and above the sparse
ranking's 256, ragged query batches, invalid given lists."""

import numpy as np
import pytest
import torch

import oracle
from cases import mixture_views, sampled_codebook, shape_ids
from helpers import assert_ranking_close

pytestmark = pytest.mark.gpu

import paper_1604_01879_b200 as gift  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402
from paper_1604_01879_b200.errors import EmptyManifest  # noqa: E402


def _build(db, C, **kw):
    cfg = gift.IndexConfig(n_views=db.shape[1], codebook_size=C.shape[0], imported=True, **kw)
    return gift.build_index_from_views(db, shape_ids(len(db)), cfg,
                                       codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")})


def _check(bundle, db, C, qs, top_k, **kw):
    ids = shape_ids(len(db))
    ref = oracle.OracleIndex(list(db), C, ids, **kw)
    got = gift.query_batch(bundle, qs, top_k=top_k)
    for q, g in zip(qs, got):
        exp, _ = ref.query(q, top_k=top_k, rerank=True)
        assert len(g) == len(exp) == min(top_k, len(db))
        assert_ranking_close([ids.index(r[0]) for r in g], [r[1] for r in g],
                             [ids.index(r[0]) for r in exp], [r[1] for r in exp])


def test_single_shape_index_and_top_k_above_n():
    views, _ = mixture_views(3, 1, 6, 32, 1, n_queries=3)
    db, qs = views[:1], views[1:]
    C = sampled_codebook(db, 2, 0)
    b = _build(db, C, ma=1, k1=3, k2=2)
    _check(b, db, C, qs, 10, ma=1, k1=3, k2=2)
    res, _ = gift.query_by_id(b, "s0000", top_k=5)
    assert [r[0] for r in res] == ["s0000"]


def test_all_zero_queries_rank_by_zero_fill():
    views, _ = mixture_views(4, 60, 5, 24, 4, n_queries=2)
    db = views[:60]
    C = sampled_codebook(db, 6, 1)
    b = _build(db, C, ma=2, k1=5, k2=3)
    qs = np.zeros((2, 5, 24), dtype=np.float32)
    got = gift.query_batch(b, qs, top_k=7)
    for g in got:  # nothing touched: every score 0, ids in order
        assert [r[0] for r in g] == shape_ids(60)[:7]
        assert all(r[1] == 0.0 for r in g)


@pytest.mark.parametrize("top_k", [255, 256, 257, 400])
def test_top_k_around_the_sparse_ranking_limit(top_k):
    views, _ = mixture_views(5, 450, 6, 32, 9, n_queries=4)
    db, qs = views[:450], views[450:]
    C = sampled_codebook(db, 12, 2)
    b = _build(db, C, ma=2, k1=6, k2=3)
    _check(b, db, C, qs, top_k, ma=2, k1=6, k2=3)


def test_ragged_query_batches_equal_single_queries():
    views, _ = mixture_views(6, 120, 6, 32, 6, n_queries=13)
    db, qs = views[:120], views[120:]
    C = sampled_codebook(db, 8, 3)
    cfg = gift.IndexConfig(n_views=6, codebook_size=8, ma=2, k1=5, k2=3, imported=True,
                           batch_size=5)
    b = gift.build_index_from_views(db, shape_ids(120), cfg,
                                    codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")})
    got = gift.query_batch(b, qs, top_k=20)  # batches of 5, 5, 3
    for q, g in zip(qs, got):
        one, _ = gift.query(b, q, top_k=20)
        assert one == g


def test_given_lists_validation():
    idx = torch.tensor([[1, 2, 2], [0, 2, 1], [0, 1, 2]], dtype=torch.int32)
    val = torch.tensor([[0.9, 0.5, 0.1]] * 3, dtype=torch.float64)
    with pytest.raises(ValueError):
        gift.build_index_from_lists(idx, val, shape_ids(3), gift.IndexConfig(k1=3, k2=2))
    with pytest.raises(EmptyManifest):
        gift.build_index_from_views(np.zeros((0, 4, 8), np.float32), [], gift.IndexConfig())
