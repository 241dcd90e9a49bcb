"""GPU: the streamed (chunked) F-IF build — config 3's path, where the
database does not fit HBM twice — is bit-identical to the in-HBM build
(matching.py:106-133 order), and an index without a storage copy scores and
ranks exactly like one with it (the scan reads only the tensor-core planes)."""

import numpy as np
import pytest
import torch

from cases import mixture_views, sampled_codebook, shape_ids

pytestmark = pytest.mark.gpu

import paper_1604_01879_b200 as gift  # noqa: E402
from paper_1604_01879_b200 import synth  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402
from paper_1604_01879_b200.errors import Unsupported  # noqa: E402

FIELDS = ("cell_off", "post_ord", "pnorm2", "feat_hi", "feat_lo", "seg_off", "seg_ord",
          "seg_pstart", "tile_off", "tile_pstart", "tile_pend", "tile_seg0", "tile_seg1",
          "shape_off", "shape_post")


def _pair(dtype, keep, chunk, N=300, V=12, d=256, K=24, zeros=True):
    views, _ = mixture_views(77, N, V, d, 9, n_queries=16, mu0=-0.2)
    db, qs = views[:N].copy(), views[N:]
    if zeros:
        db[3, 5:] = 0.0  # ragged view sets (zero views are not stored)
        db[17, :] = 0.0  # a shape with no stored view at all
    C = sampled_codebook(db, K, 4)
    cfg = gift.IndexConfig(n_views=V, codebook_size=K, ma=2, k1=6, k2=3, imported=True,
                           similarity="gaussian", storage_dtype=dtype)
    ids = shape_ids(N)
    cbs = {"A": Codebook(C, "A"), "B": Codebook(C, "B")}
    full = gift.build_index_from_views(db, ids, cfg, codebooks=cbs)
    Xd = torch.from_numpy(db).cuda().to(cfg.torch_storage)
    streamed = gift.build_index_streamed(lambda s0, s1: Xd[s0:s1].float(), ids, V, d, cfg,
                                         codebooks=cbs, chunk=chunk, keep_features=keep,
                                         self_join_batch=64)
    return full, streamed, qs


@pytest.mark.parametrize("dtype,keep,chunk", [("float32", True, 64), ("float32", False, 37),
                                              ("float16", False, 100)])
def test_streamed_build_bit_identical(dtype, keep, chunk):
    full, st, qs = _pair(dtype, keep, chunk)
    a, b = full.fifs["A"].dev, st.fifs["A"].dev
    assert a.P == b.P and a.S == b.S and a.T == b.T
    for name in FIELDS:
        x, y = getattr(a, name), getattr(b, name)
        if x is None:
            assert y is None, name
            continue
        assert torch.equal(x, y), name
    if keep or dtype == "float16":
        assert torch.equal(a.feat, b.feat)
    else:
        assert b.feat is None
        with pytest.raises(Unsupported):
            st.fifs["A"].entry_features
    # self-join -> raw activations and S-IF identical
    ra, rb = full.raw_activations["A"], st.raw_activations["A"]
    for x, y in zip(ra, rb):
        np.testing.assert_array_equal(np.asarray(x.indices), np.asarray(y.indices))
        np.testing.assert_array_equal(np.asarray(x.values), np.asarray(y.values))
    sa, sb = full.sif.dev, st.sif.dev
    for name in ("e_off", "e_ord", "e_val", "norms"):
        assert torch.equal(getattr(sa, name), getattr(sb, name)), name
    # queries: identical rankings and scores
    ga = gift.query_batch(full, qs, top_k=20, rerank=True)
    gb = gift.query_batch(st, qs, top_k=20, rerank=True)
    assert ga == gb


def test_streamed_query_by_id_from_planes():
    full, st, _ = _pair("float32", False, 50)
    fa, fb = full.fifs["A"], st.fifs["A"]
    m_full = fa.shape_matrix(5)
    m_pl = fb.shape_matrix(5)
    np.testing.assert_allclose(m_pl, m_full, rtol=2.0 ** -20, atol=1e-30)


def test_block_mixture_regenerates_identically():
    w = synth.Workload("t", 600, 4, 64, 7, 16, 2, 0.5, 10, 4, 10, 40, 16, -0.2)
    mix = synth.BlockMixture(w, 5, torch.device("cuda", 0), block=64)
    a = mix.rows(0, 600)
    b = torch.cat([mix.rows(s, min(600, s + 97)) for s in range(0, 600, 97)])
    assert torch.equal(a, b)
    C = synth.sample_centroids_rows(mix, 16, 3)
    ref = synth.sample_centroids(a, 16, 3)
    assert torch.equal(C, ref)
