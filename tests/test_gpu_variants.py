"""GPU: kernel-variant selection through explicit flags, the fp16-exact query
shortcut of the scan, and the k2 edge cases of the re-rank (k2 > 8 takes the
dense neighbour path; k2 = 64 fills the mean activation's neighbour table)."""

import numpy as np
import pytest
import torch

import oracle
from cases import mixture_views, sampled_codebook, shape_ids
from helpers import RTOL, assert_ranking_close

pytestmark = pytest.mark.gpu

import paper_1604_01879_b200 as gift  # noqa: E402
from paper_1604_01879_b200 import engine as eg  # noqa: E402
from paper_1604_01879_b200 import matching as mt  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402
from paper_1604_01879_b200.errors import Unsupported  # noqa: E402


def dev():
    return torch.device("cuda", 0)


@pytest.mark.parametrize("pair", ["off", "on"])
@pytest.mark.parametrize("storage", ["float16", "float32"])
def test_fp16_exact_queries_skip_lo_plane_bit_identical(storage, pair):
    """Queries whose values are exactly fp16 have an all-zero lo plane: the
    scan then drops the b2 operand (single CTA: one N = n MMA per k-step;
    fp16-storage CTA pairs: N = 256 probe columns per item instead of
    [b1 | b2] over 128).  A batch with one non-fp16 value elsewhere takes the
    full [b1 | b2] path; the fp16-exact queries must score bit-identically in
    both batches, and match the widened oracle."""
    views, _ = mixture_views(31, 240, 20, 256, 12, n_queries=5)
    db = views[:240].astype(np.float16 if storage == "float16" else np.float32)
    q16 = views[240:].astype(np.float16).astype(np.float32)  # fp16-exact
    C = sampled_codebook(db.astype(np.float32), 24, 2)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev()), Codebook(C), shape_ids(240))
    fif.dev.set_variant(pair=pair)
    other = views[240:241].copy()
    other[0, 0, 7] += np.float32(1e-6)  # not representable in fp16: lo plane non-zero
    for sim in ("gaussian", "cosine"):
        a = mt.query_fif_batch(fif, q16, 1, sim).cpu().numpy()
        b = mt.query_fif_batch(fif, np.concatenate([q16, other]), 1, sim).cpu().numpy()[:5]
        np.testing.assert_array_equal(a, b)
        dbw = db.astype(np.float32)
        assign = oracle.quantize_many(C, dbw.reshape(-1, 256), 1).reshape(240, 20)
        ref = oracle.build_fif(list(dbw), C, assign=assign)
        for q, g in zip(q16, a):
            e = oracle.query_fif(ref, q, 1, sim, cells=oracle.quantize_many(C, q.astype(np.float64), 1))
            np.testing.assert_allclose(g, e, rtol=RTOL, atol=1e-9)
    fif.dev.set_variant()


def _oracle_rank(db, qs, C, ids, ma, k1, k2, top_k):
    ref = oracle.OracleIndex(list(db), C, ids, ma=ma, k1=k1, k2=k2)
    return [ref.query(q, top_k=top_k, rerank=True)[0] for q in qs]


@pytest.mark.parametrize("k1,k2", [(10, 10), (12, 64), (3, 9)])
def test_large_k2_against_oracle(k1, k2):
    """k2 above the reduce's candidate limit (8) runs through the dense
    scores; k2 = 64 = the mean kernel's neighbour-table size."""
    N, V, d, K = 180, 6, 32, 10
    views, _ = mixture_views(41 + k2, N, V, d, 5, n_queries=4)
    db, qs = views[:N], views[N:]
    ids = shape_ids(N)
    C = sampled_codebook(db, K, 3)
    cfg = gift.IndexConfig(n_views=V, codebook_size=K, ma=2, k1=k1, k2=k2, imported=True)
    bundle = gift.build_index_from_views(db, ids, cfg,
                                         codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")})
    got = gift.query_batch(bundle, qs, top_k=25)
    exp = _oracle_rank(db, qs, C, ids, 2, k1, k2, 25)
    for g, e in zip(got, exp):
        assert_ranking_close([ids.index(r[0]) for r in g], [r[1] for r in g],
                             [ids.index(r[0]) for r in e], [r[1] for r in e])


def test_kernel_limits_rejected_at_config():
    with pytest.raises(Unsupported):
        gift.IndexConfig(k1=20, k2=65)
    with pytest.raises(Unsupported):
        gift.IndexConfig(k1=100, k2=11)


def test_drain_interval_flag_validated():
    views, _ = mixture_views(5, 40, 4, 64, 3, n_queries=2)
    C = sampled_codebook(views[:40], 8, 1)
    fif = mt.build_fif_from_tensor(torch.from_numpy(views[:40]).to(dev()), Codebook(C),
                                   shape_ids(40))
    base = mt.query_fif_batch(fif, views[40:], 2, "gaussian").cpu().numpy()
    for kb in (1, 2, 3):
        fif.dev.set_variant(drain_kb=kb)
        np.testing.assert_allclose(mt.query_fif_batch(fif, views[40:], 2, "gaussian").cpu().numpy(),
                                   base, rtol=RTOL)
    fif.dev.set_variant(drain_kb=17)
    with pytest.raises(ValueError):
        mt.query_fif_batch(fif, views[40:], 2, "gaussian")
    fif.dev.set_variant()


@pytest.mark.parametrize("storage", ["float16", "float32"])
def test_scan_variants_many_probes_per_cell(storage):
    """Cells with hundreds of probes (several probe tiles per posting tile,
    items of N = 64 and 128 interleaved), so the two epilogue groups run
    different items at once: every scan variant (single CTA / CTA pairs,
    drain interval 4 / 8 / 16, fp16-exact and general queries) stays within
    the contract of the f64 oracle."""
    rng = np.random.default_rng(17)
    views, _ = mixture_views(71, 1500, 8, 256, 6, n_queries=72)
    db = views[:1500].astype(np.float16 if storage == "float16" else np.float32)
    C = sampled_codebook(db.astype(np.float32), 5, 3)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev()), Codebook(C), shape_ids(1500))
    dbw = db.astype(np.float32)
    assign = oracle.quantize_many(C, dbw.reshape(-1, 256), 1).reshape(1500, 8)
    ref_fif = oracle.build_fif(list(dbw), C, assign=assign)
    for qname, qs in (("q16", views[1500:].astype(np.float16).astype(np.float32)),
                      ("q32", views[1500:])):
        ref = np.stack([oracle.query_fif(ref_fif, q, 1, "gaussian",
                                         cells=oracle.quantize_many(C, q.astype(np.float64), 1))
                        for q in qs])
        for pair in ("off", "on"):
            for kb in (4, 8, 16):
                fif.dev.set_variant(pair=pair, drain_kb=kb)
                got = mt.query_fif_batch(fif, qs, 1, "gaussian").cpu().numpy()
                np.testing.assert_allclose(got, ref, rtol=RTOL, atol=1e-12,
                                           err_msg=f"{storage} {qname} pair={pair} drain={kb}")
    fif.dev.set_variant()
    del rng


@pytest.mark.parametrize("sim", ["gaussian", "cosine"])
def test_dense_cells_probe_major_scan(sim):
    """fp16 storage with cells probed by >= 192 query views in one batch: the
    dense cells run on the probe-major CTA-pair scan (fif_scan_dense.cu; odd
    posting-tile counts, probe counts not a multiple of 256, CTAs without
    valid probes), the others on the single-CTA scan.  Scores match the
    widened f64 oracle and equal the posting-major scan of every cell
    (dense="off") bit for bit; a batch with a non-fp16 query
    value takes no dense split and scores the fp16-exact queries the same."""
    views, _ = mixture_views(83, 1600, 8, 256, 5, n_queries=150)
    db = views[:1600].astype(np.float16)
    qs = views[1600:].astype(np.float16).astype(np.float32)
    C = sampled_codebook(db.astype(np.float32), 6, 4)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev()), Codebook(C), shape_ids(1600))
    dbw = db.astype(np.float32)
    assign = oracle.quantize_many(C, dbw.reshape(-1, 256), 1).reshape(1600, 8)
    ref_fif = oracle.build_fif(list(dbw), C, assign=assign)
    qcells = oracle.quantize_many(C, qs.reshape(-1, 256).astype(np.float64), 1).reshape(150, 8, 1)
    counts = np.bincount(qcells.ravel(), minlength=6)
    assert counts.max() >= 192, counts  # some cells take the dense scan
    ref = np.stack([oracle.query_fif(ref_fif, q, 1, sim, cells=c) for q, c in zip(qs, qcells)])
    got = mt.query_fif_batch(fif, qs, 1, sim).cpu().numpy()
    np.testing.assert_allclose(got, ref, rtol=RTOL, atol=1e-12, err_msg="dense")
    for kw in ({"sched": "static"}, {"drain_kb": 4}, {"drain_kb": 16}):
        fif.dev.set_variant(**kw)  # static item stride; drain intervals
        np.testing.assert_allclose(mt.query_fif_batch(fif, qs, 1, sim).cpu().numpy(), ref,
                                   rtol=RTOL, atol=1e-12, err_msg=str(kw))
    fif.dev.set_variant(dense="off")
    off = mt.query_fif_batch(fif, qs, 1, sim).cpu().numpy()
    np.testing.assert_allclose(off, ref, rtol=RTOL, atol=1e-12, err_msg="dense off")
    np.testing.assert_array_equal(got, off)  # same MMA sums, same epilogue arithmetic
    fif.dev.set_variant()
    other = views[1600:1601].copy()
    other[0, 0, 3] += np.float32(1e-6)  # lo plane non-zero: no dense split
    mixed = mt.query_fif_batch(fif, np.concatenate([qs, other]), 1, sim).cpu().numpy()[:150]
    np.testing.assert_allclose(mixed, ref, rtol=RTOL, atol=1e-12, err_msg="mixed batch")


@pytest.mark.parametrize("storage", ["float32", "float16"])
def test_graphed_query_equals_eager(storage):
    """The whole query pipeline captured in a CUDA graph (GraphedQuery) and
    replayed on new batches returns exactly eng.run's rankings and scores
    (every kernel graph-safe: no host synchronisation, device-side plan
    sizes); fp16 storage includes dense cells (the probe-major scan)."""
    N, V, d, K = 600, 8, 64, 3
    views, _ = mixture_views(91, N, V, d, 5, n_queries=150)
    db = views[:N].astype(np.float16 if storage == "float16" else np.float32)
    qs = views[N:].astype(np.float16).astype(np.float32)
    C = sampled_codebook(db.astype(np.float32), K, 2)
    cfg = gift.IndexConfig(n_views=V, codebook_size=K, ma=1, k1=6, k2=3, imported=True,
                           storage_dtype=storage, similarity="gaussian")
    bundle = gift.build_index_from_views(db, shape_ids(N), cfg,
                                         codebooks={"A": Codebook(C, "A"),
                                                    "B": Codebook(C, "B")})
    eng = bundle.engine
    Q = torch.from_numpy(qs).to(dev())
    batches = [Q[i:i + 50].contiguous() for i in (0, 50, 100)]
    gq = gift.GraphedQuery(eng, batches[0], top_k=20)
    for b in batches + batches[::-1]:
        ei, ev = eng.run(b, top_k=20, rerank=True)
        gi, gv = gq(b)
        torch.cuda.synchronize()
        assert torch.equal(ei, gi) and torch.equal(ev, gv)


def test_graph_survives_scratch_regrowth_on_its_stream():
    """A bigger eager batch on the graph's own stream regrows that stream's
    scratch (grow-only caches); the buffers the graph captured stay alive, so
    later replays still equal eager runs."""
    N, V, d, K = 400, 8, 64, 3
    views, _ = mixture_views(92, N, V, d, 5, n_queries=160)
    db, qs = views[:N], views[N:]
    C = sampled_codebook(db, K, 2)
    cfg = gift.IndexConfig(n_views=V, codebook_size=K, ma=1, k1=6, k2=3, imported=True)
    bundle = gift.build_index_from_views(db, shape_ids(N), cfg,
                                         codebooks={"A": Codebook(C, "A"),
                                                    "B": Codebook(C, "B")})
    eng = bundle.engine
    Q = torch.from_numpy(qs).to(dev())
    small, big = Q[:20].contiguous(), Q[20:160].contiguous()
    gq = gift.GraphedQuery(eng, small, top_k=15)
    with torch.cuda.stream(gq.stream):
        eng.run(big, top_k=15, rerank=True)  # regrows the stream's scratch
    for b in (Q[40:60].contiguous(), small):
        ei, ev = eng.run(b, top_k=15, rerank=True)
        gi, gv = gq(b)
        torch.cuda.synchronize()
        assert torch.equal(ei, gi) and torch.equal(ev, gv)
