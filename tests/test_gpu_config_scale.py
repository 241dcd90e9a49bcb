"""GPU parity at BASELINE.json's own config sizes.

* C1 exactly as specified (N=1,000 x V=64 x d=256, K=64, ma=1, k1=10, k2=4,
  100 queries, top-50): cosine mode against goldens the REFERENCE produced
  (tests/golden/make_golden.py c1), gaussian mode against the oracle.
* C2 (N=10,000 x V=64 x d=4,096, K=256, ma=2, gaussian sigma=0.5, top-100):
  the whole database quantized and laid out by the oracle on the host
  (bit-exact lists), its full f64 self-join (raw activations), the S-IF,
  and 64 sampled queries scored against all 10,000 shapes and ranked.
* C5 (given top-50 lists, k1=50, k2=4, top-100) at N=50,000 with 1,024
  queries through both S-IF query implementations (accumulator rows and the
  sort-based one).

Relative score errors (max, p99.99) are recorded through
helpers.record_parity ($GIFT_PARITY_OUT; committed under profiles/)."""

import gc

import numpy as np
import pytest
import torch

import oracle
from cases import C1, c1_inputs
from conftest import load_golden
from helpers import (RTOL, assert_ranking_close, assert_topk_rows_close, record_parity,
                     rel_err_stats, unpack_acts)
from oracle import scale

pytestmark = pytest.mark.gpu

import paper_1604_01879_b200 as gift  # noqa: E402
from paper_1604_01879_b200 import _native as nat  # noqa: E402
from paper_1604_01879_b200 import matching as mt  # noqa: E402
from paper_1604_01879_b200 import synth  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook, quantize_batch  # noqa: E402

SEED = 20160407  # bench.py's workload seed


@pytest.fixture(autouse=True)
def _free_hbm():
    """Config-scale indexes take up to ~130 GB: release the previous test's
    (reference cycles, the thread's scan workspaces, cached blocks) first."""
    gc.collect()
    mt.release_workspaces()
    torch.cuda.empty_cache()
    yield
    gc.collect()
    mt.release_workspaces()
    torch.cuda.empty_cache()


def dev():
    return torch.device("cuda", 0)


def _bundle(db, ids, C, **cfg):
    config = gift.IndexConfig(imported=True, **cfg)
    return gift.build_index_from_views(db, ids, config,
                                       codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")})


def _gpu_lists(bundle):
    f = bundle.fifs["A"].dev
    return f.cell_off.cpu().numpy(), f.post_ord.cpu().numpy()


def _raw_rows(bundle):
    return [(i, v) for i, v, _n in bundle.raw_activations["A"].rows.to_host()]


def _nbrs_from_raw(raw_rows, k2):
    """top_neighbors (rerank.py:78-87) of a self-join row, read off its raw
    activation: the top-k1 entries by (score desc, ordinal asc), zeros
    already dropped, k1 >= k2."""
    out = []
    for idx, val in raw_rows:
        o = np.lexsort((idx, -val))[:k2]
        out.append([int(idx[j]) for j in o])
    return out


def _oracle_acts(rows):
    return [oracle.make_activation(i, v) for i, v in rows]


def _check_sif_against(bundle, final_ref, sif_ref):
    """The device S-IF equals the oracle's transpose (rerank.py:187-208)
    bit for bit: ordinals ascending per entry, values and norms exact."""
    d = bundle.sif.dev
    off = d.e_off.cpu().numpy()
    e_ord = d.e_ord.cpu().numpy()
    e_val = d.e_val.cpu().numpy()
    np.testing.assert_array_equal(d.norms.cpu().numpy(), sif_ref.norms)
    ref_len = np.array([len(o) for o in sif_ref.entry_ordinals])
    np.testing.assert_array_equal(np.diff(off), ref_len)
    np.testing.assert_array_equal(e_ord, np.concatenate(sif_ref.entry_ordinals))
    np.testing.assert_array_equal(e_val, np.concatenate(sif_ref.entry_values))


def _rank_ids(res, ids_index):
    return [ids_index[r[0]] for r in res], [r[1] for r in res]


# ------------------------------------------------------------------ C1
def test_c1_exact_config_cosine_against_reference():
    db, qs, C, ids = c1_inputs()
    g = load_golden("c1.npz")
    np.testing.assert_array_equal(C, g["C"])
    b = _bundle(db, ids, C, n_views=C1["V"], codebook_size=C1["K"], ma=C1["ma"], k1=C1["k1"],
                k2=C1["k2"])
    cell_off, post_ord = _gpu_lists(b)
    np.testing.assert_array_equal(np.diff(cell_off), g["fif_len"])  # lists bit-exact
    np.testing.assert_array_equal(post_ord, g["fif_ord"])
    raw_ref = [(i, v) for i, v, _n in unpack_acts(g, "raw")]
    swaps = assert_topk_rows_close(_raw_rows(b), raw_ref)
    sc = mt.query_fif_batch(b.fifs["A"], qs, C1["ma"]).cpu().numpy()
    st = rel_err_stats(sc, g["q_fif_scores"])
    record_parity("c1", "fif_scores_cosine_vs_reference", {**st, "raw_swaps": swaps})
    assert st["max"] <= RTOL and st["zero_mismatch"] == 0
    rs = np.stack([gift.rerank_scores(b, {"A": s, "B": s}) for s in g["q_fif_scores"]])
    st = rel_err_stats(rs, g["q_rerank_scores"])
    record_parity("c1", "rerank_scores_cosine_vs_reference", st)
    assert st["max"] <= RTOL
    pos = {s: i for i, s in enumerate(ids)}
    for rerank, tag in ((True, "rr"), (False, "nr")):
        got = gift.query_batch(b, qs, top_k=C1["top_k"], rerank=rerank)
        for qi in range(len(qs)):
            gi, gs = _rank_ids(got[qi], pos)
            assert_ranking_close(gi, gs, g[f"q_{tag}_ids"][qi], g[f"q_{tag}_scores"][qi])
        for j, i in enumerate(range(0, len(ids), 125)):
            res, _ = gift.query_by_id(b, ids[i], top_k=C1["top_k"], rerank=rerank)
            gi, gs = _rank_ids(res, pos)
            assert_ranking_close(gi, gs, g[f"id_{tag}_ids"][j], g[f"id_{tag}_scores"][j])


def test_c1_exact_config_gaussian_against_oracle():
    db, qs, C, ids = c1_inputs()
    kw = dict(ma=C1["ma"], k1=C1["k1"], k2=C1["k2"])
    b = _bundle(db, ids, C, n_views=C1["V"], codebook_size=C1["K"], similarity="gaussian",
                sigma=C1["sigma"], **kw)
    orc = scale.OracleCsrIndex.from_views(db, C, similarity="gaussian", sigma=C1["sigma"], **kw)
    cell_off, post_ord = _gpu_lists(b)
    np.testing.assert_array_equal(cell_off, orc.cell_off)
    np.testing.assert_array_equal(post_ord, orc.post_ord)
    raw_gpu = _raw_rows(b)
    swaps = assert_topk_rows_close(raw_gpu, [(a.idx, a.val) for a in orc.raw])
    q_sc = mt.query_fif_batch(b.fifs["A"], qs, C1["ma"], "gaussian", C1["sigma"]).cpu().numpy()
    ref_sc = orc.scores(qs)
    st = rel_err_stats(q_sc, ref_sc)
    record_parity("c1", "fif_scores_gaussian_vs_oracle", {**st, "raw_swaps": swaps})
    assert st["max"] <= RTOL and st["zero_mismatch"] == 0
    # S-IF of the device's own raw activations (mean + aggregate + transpose, exact)
    raw_acts = _oracle_acts(raw_gpu)
    final, sif = scale.build_context(raw_acts, _nbrs_from_raw(raw_gpu, C1["k2"]))
    _check_sif_against(b, final, sif)
    pos = {s: i for i, s in enumerate(ids)}
    got = gift.query_batch(b, qs, top_k=C1["top_k"])
    for qi, q in enumerate(qs):
        fin = scale.rerank_query(raw_acts, sif, ref_sc[qi], C1["k2"])
        order = scale.rank_final(fin, ids, "query", C1["top_k"])
        gi, gs = _rank_ids(got[qi], pos)
        assert_ranking_close(gi, gs, order, fin[order])


# ------------------------------------------------------------------ C2
@pytest.fixture(scope="class")
def c2():
    w = synth.WORKLOADS["c2"]
    db, qs, _ = synth.mixture(w, SEED, dev())  # the bench's own workload (device generator)
    C = synth.sample_centroids(db, w.K, SEED + 1).cpu().numpy()
    ids = synth.shape_ids(w.n_shapes)
    b = _bundle(db, ids, C, n_views=w.n_views, codebook_size=w.K, ma=w.ma, k1=w.k1, k2=w.k2,
                similarity="gaussian", sigma=w.sigma, batch_size=w.batch)
    sel = np.sort(np.random.default_rng(64).choice(qs.shape[0], 64, replace=False))
    q = qs[torch.from_numpy(sel).to(dev())].contiguous()
    db_h = db.cpu().numpy()
    orc = scale.OracleCsrIndex.from_views(db_h, C, w.ma, w.k1, w.k2, "gaussian", w.sigma)
    yield dict(w=w, db=db, b=b, q=q, q_h=q.cpu().numpy(), C=C, ids=ids, orc=orc)
    del db, b
    torch.cuda.empty_cache()


class TestC2:
    """The C2 index lives for these three tests only (class-scoped fixture)."""

    def test_c2_lists_bit_exact(self, c2):
        orc, b = c2["orc"], c2["b"]
        cell_off, post_ord = _gpu_lists(b)
        np.testing.assert_array_equal(cell_off, orc.cell_off)
        np.testing.assert_array_equal(post_ord, orc.post_ord)
        d = c2["w"].dim
        rows = torch.from_numpy(orc.rows).to(dev())
        assert torch.equal(b.fifs["A"].dev.feat, c2["db"].reshape(-1, d)[rows])
        # the 64 queries' multiple assignment (ma = 2), bit-exact
        got = quantize_batch(Codebook(c2["C"]), c2["q"].reshape(-1, d), 2)
        ref = scale.quantize_many_mt(c2["C"], c2["q_h"].reshape(-1, d), 2)
        np.testing.assert_array_equal(got, ref)


    def test_c2_scores_64_queries_vs_oracle(self, c2):
        w, orc = c2["w"], c2["orc"]
        got = mt.query_fif_batch(c2["b"].fifs["A"], c2["q"], w.ma, "gaussian", w.sigma).cpu().numpy()
        ref = orc.scores(c2["q_h"])
        st = rel_err_stats(got, ref)
        record_parity("c2", "fif_scores_gaussian_vs_oracle_64q_x_10k", st)
        assert st["max"] <= RTOL and st["zero_mismatch"] == 0


    def test_c2_scores_64_queries_cosine_and_f64_vs_oracle(self, c2):
        """The same index and 64 queries through the cosine kernel (the
        reference's own similarity, matching.py:158) and through the f64 path
        (precision="f64", 8 queries), against the oracle's f64 scores."""
        w, orc = c2["w"], c2["orc"]
        B, V, d = c2["q_h"].shape
        qc = scale.quantize_many_mt(c2["C"], c2["q_h"].reshape(B * V, d), w.ma).reshape(B, V, w.ma)
        qc = np.where(c2["q_h"].any(axis=2)[:, :, None], qc, -1)
        ref = scale.fif_scores_many(orc.cell_off, orc.post_ord, orc.feat_rows, c2["q_h"], qc,
                                    w.n_shapes, "cosine")
        got = mt.query_fif_batch(c2["b"].fifs["A"], c2["q"], w.ma, "cosine").cpu().numpy()
        st = rel_err_stats(got, ref)
        record_parity("c2", "fif_scores_cosine_vs_oracle_64q_x_10k", st)
        assert st["max"] <= RTOL and st["zero_mismatch"] == 0
        got64 = mt.query_fif_batch(c2["b"].fifs["A"], c2["q"][:8], w.ma, "cosine",
                                   precision="f64").cpu().numpy()
        np.testing.assert_allclose(got64, ref[:8], rtol=1e-12, atol=1e-15)
        record_parity("c2", "fif_scores_cosine_f64_path_vs_oracle_8q_x_10k",
                      rel_err_stats(got64, ref[:8]))

    def test_c2_self_join_sif_and_rankings(self, c2):
        w, orc, b, ids = c2["w"], c2["orc"], c2["b"], c2["ids"]
        raw_gpu = _raw_rows(b)
        swaps = assert_topk_rows_close(raw_gpu, [(a.idx, a.val) for a in orc.raw])
        vals = np.concatenate([v for _i, v in raw_gpu])
        ref_vals = np.concatenate([a.val for a in orc.raw])
        st = rel_err_stats(vals, ref_vals) if swaps == 0 else {"n": int(len(vals))}
        record_parity("c2", "self_join_raw_activations_vs_oracle", {**st, "raw_swaps": swaps,
                                                                     "rows": len(raw_gpu)})
        raw_acts = _oracle_acts(raw_gpu)
        final, sif = scale.build_context(raw_acts, _nbrs_from_raw(raw_gpu, w.k2))
        _check_sif_against(b, final, sif)
        ref_sc = orc.scores(c2["q_h"])
        got = gift.query_batch(b, c2["q"], top_k=w.top_k)
        pos = {s: i for i, s in enumerate(ids)}
        agree = 0
        for qi in range(ref_sc.shape[0]):
            fin = scale.rerank_query(raw_acts, sif, ref_sc[qi], w.k2)
            order = scale.rank_final(fin, ids, "query", w.top_k)
            gi, gs = _rank_ids(got[qi], pos)
            assert_ranking_close(gi, gs, order, fin[order])
            # fully independent: the oracle's own raw activations and S-IF
            fin2 = scale.rerank_query(orc.raw, orc.sif, ref_sc[qi], w.k2)
            agree += int(list(scale.rank_final(fin2, ids, "query", w.top_k)) == gi)
        record_parity("c2", "rankings_top100_64q", {"queries": int(ref_sc.shape[0]),
                                                    "identical_to_independent_oracle": agree})


# ------------------------------------------------------------------ C5
def _c5_oracle(idx_h, val_h, k1, k2):
    """index.py:196-218 on given best-first lists: build_activation keeps the
    first k1 positive entries, top_neighbors the first k2 (rerank.py:64-87)."""
    raw = [oracle.make_activation(i[:k1], v[:k1]) for i, v in zip(idx_h, val_h)]
    nbrs = [[int(j) for j, x in zip(i[:k2], v[:k2]) if x > 0.0] for i, v in zip(idx_h, val_h)]
    final, sif = scale.build_context(raw, nbrs)
    return raw, final, sif


@pytest.mark.parametrize("n_shapes", [50_000])
def test_c5_given_lists_against_oracle(n_shapes):
    c = synth.C5
    # communities of ~500 members as at N = 1M (45 in-community picks per list)
    idx, val = synth.community_lists(SEED, dev(), n_shapes=n_shapes,
                                     communities=max(1, n_shapes // 500))
    ids = synth.shape_ids(n_shapes)
    cfg = gift.IndexConfig(k1=c["list_len"], k2=c["k2"], imported=True, batch_size=c["batch"])
    b = gift.build_index_from_lists(idx, val, ids, cfg)
    idx_h, val_h = idx.cpu().numpy().astype(np.int64), val.cpu().numpy()
    raw, final, sif = _c5_oracle(idx_h, val_h, c["list_len"], c["k2"])
    got_raw = b.raw_activations["A"].rows.to_host()
    for (gi, gv, gn), a in zip(got_raw, raw):
        np.testing.assert_array_equal(gi, a.idx)
        np.testing.assert_array_equal(gv, a.val)
        assert gn == a.norm
    _check_sif_against(b, final, sif)
    rows = np.sort(np.random.default_rng(5).choice(n_shapes, 1024, replace=False))
    eng = b.engine
    r = torch.from_numpy(rows).to(dev())
    outs = {}
    for mode, flags in (("rows", nat.SIF_ROWS), ("sort", nat.SIF_SORT),
                        ("bucket", nat.SIF_BUCKET)):
        eng.sif.query_flags = flags
        gi, gv = [], []
        for s in range(0, len(rows), c["batch"]):
            rr = r[s:s + c["batch"]]
            i2, v2 = eng.rerank_lists(idx[rr], val[rr], top_k=c["top_k"],
                                      self_local=rr.to(torch.int32))
            gi.append(i2.cpu().numpy())
            gv.append(v2.cpu().numpy())
        outs[mode] = (np.concatenate(gi), np.concatenate(gv))
    eng.sif.query_flags = 0
    for mode in ("sort", "bucket"):
        np.testing.assert_array_equal(outs["rows"][0], outs[mode][0])
        np.testing.assert_array_equal(outs["rows"][1], outs[mode][1])
    gi, gv = outs["rows"]
    for n, q in enumerate(rows):
        nb = [int(j) for j, x in zip(idx_h[q][:c["k2"]], val_h[q][:c["k2"]]) if x > 0.0]
        f = oracle.mean_activation(raw, nb)
        fin = oracle.query_sif(sif, oracle.aggregate(f, f, 0.5))
        order = scale.rank_final(fin, ids, ids[q], c["top_k"])
        np.testing.assert_array_equal(gi[n], order)  # f64 in the reference's order: exact
        np.testing.assert_array_equal(gv[n], fin[order])
    record_parity("c5", f"rankings_top100_{len(rows)}q_n{n_shapes}",
                  {"queries": len(rows), "sif_postings": int(sum(len(o) for o in sif.entry_ordinals)),
                   "exact": True})


# ------------------------------------------------------------------ C3 / C4 (sampled)
def _raw_arrays(bundle):
    r = bundle.raw_activations["A"].rows
    return r.idx.cpu().numpy(), r.val.cpu().numpy(), r.cnt.cpu().numpy()


def _nbrs_from_raw_arrays(ri, rv, rc, k2):
    """top_neighbors of every self-join row read off its raw activation
    (best k2 by value desc, ordinal asc; zeros already dropped), [N, k2]."""
    k1 = ri.shape[1]
    valid = np.arange(k1)[None, :] < rc[:, None]
    v = np.where(valid, rv, -np.inf)
    i = np.where(valid, ri, np.iinfo(np.int32).max)
    order = np.lexsort((i, -v), axis=1)[:, :k2]
    nb = np.take_along_axis(ri, order, axis=1).astype(np.int64)
    ok = np.take_along_axis(valid, order, axis=1)
    return np.where(ok, nb, -1)


def _acts_of(ri, rv, rc, rows):
    return {int(j): oracle.Act(ri[j, :rc[j]].astype(np.int64), rv[j, :rc[j]], 0.0) for j in rows}


def _rerank_from_arrays(ri, rv, rc, sif, scores, k2):
    """index.py:249-258 with the raw activations given as arrays."""
    nb = oracle.top_neighbors(scores, k2)
    acts = _acts_of(ri, rv, rc, nb)
    f = oracle.mean_activation(acts, nb)
    return oracle.query_sif(sif, oracle.aggregate(f, f, 0.5))


def _check_scale_rerank(name, b, w, ref_sc, q_dev, ids):
    """S-IF of the device's raw activations (vectorized oracle, exact) and
    the final top-k of the sampled queries against the oracle's re-rank."""
    ri, rv, rc = _raw_arrays(b)
    nbr = _nbrs_from_raw_arrays(ri, rv, rc, w.k2)
    _fi, _fv, _fc, norms, sif = scale.build_context_arrays(ri, rv, rc, nbr)
    d = b.sif.dev
    np.testing.assert_array_equal(d.norms.cpu().numpy(), norms)
    np.testing.assert_array_equal(np.diff(d.e_off.cpu().numpy()),
                                  [len(o) for o in sif.entry_ordinals])
    np.testing.assert_array_equal(d.e_ord.cpu().numpy(), np.concatenate(sif.entry_ordinals))
    np.testing.assert_array_equal(d.e_val.cpu().numpy(), np.concatenate(sif.entry_values))
    got = gift.query_batch(b, q_dev, top_k=w.top_k)
    pos = {s: i for i, s in enumerate(ids)}
    for qi in range(ref_sc.shape[0]):
        fin = _rerank_from_arrays(ri, rv, rc, sif, ref_sc[qi], w.k2)
        order = scale.rank_final(fin, ids, "query", w.top_k)
        gi, gs = _rank_ids(got[qi], pos)
        assert_ranking_close(gi, gs, order, fin[order])
    record_parity(name, f"rankings_top{w.top_k}_{ref_sc.shape[0]}q", {"queries": ref_sc.shape[0]})


def test_c4_sampled_queries_against_oracle():
    """Config 4 at full size: 1M shapes x 20 views x d=1024 fp16, Zipf cells
    over K=4096.  Sampled DB shapes' lists and the 16 queries' assignments
    bit-exact; 16 queries scored against all 1M shapes by the oracle over the
    (verified) lists; 8 DB shapes' self-join rows; the S-IF; the rankings."""
    w = synth.WORKLOADS["c4"]
    db, qs, Ct = synth.zipf_mixture(w, SEED, dev())
    C = Ct.cpu().numpy()
    ids = synth.shape_ids(w.n_shapes)
    b = _bundle(db, ids, C, n_views=w.n_views, codebook_size=w.K, ma=w.ma, k1=w.k1, k2=w.k2,
                similarity="gaussian", sigma=w.sigma, storage_dtype=w.storage,
                batch_size=w.batch)
    rng = np.random.default_rng(4)
    samp = np.sort(rng.choice(w.n_shapes, 200, replace=False))
    samp_views = db[torch.from_numpy(samp).to(dev())].float().cpu().numpy()
    del db
    torch.cuda.empty_cache()
    f = b.fifs["A"].dev
    cell_off, post_ord = f.cell_off.cpu().numpy(), f.post_ord.cpu().numpy()
    shape_off, shape_post = f.shape_off.cpu().numpy(), f.shape_post.cpu().numpy()
    feat = f.feat.cpu().numpy()  # fp16 [P, d]
    # (1) lists: each sampled shape's postings are its non-zero views in
    # cell order (view order inside a cell), under the oracle's cells
    cells = scale.quantize_many_mt(C, samp_views.reshape(-1, w.dim), 1)[:, 0].reshape(200, -1)
    for k, i in enumerate(samp):
        nz = samp_views[k].any(axis=1)
        o = np.argsort(np.where(nz, cells[k], 1 << 30), kind="stable")[:int(nz.sum())]
        p = shape_post[shape_off[i]:shape_off[i + 1]]
        np.testing.assert_array_equal(np.searchsorted(cell_off, p, side="right") - 1, cells[k][o])
        np.testing.assert_array_equal(feat[p].astype(np.float32), samp_views[k][o])
    # (2) the 16 queries: assignment bit-exact, scores vs the oracle
    sel = np.sort(rng.choice(qs.shape[0], 16, replace=False))
    q = qs[torch.from_numpy(sel).to(dev())].contiguous()
    q_h = q.cpu().numpy()
    qc = scale.quantize_many_mt(C, q_h.reshape(-1, w.dim), w.ma)
    np.testing.assert_array_equal(quantize_batch(Codebook(C), q.reshape(-1, w.dim), w.ma), qc)
    got = mt.query_fif_batch(b.fifs["A"], q, w.ma, "gaussian", w.sigma).cpu().numpy()
    ref = scale.fif_scores_many(cell_off, post_ord, lambda a, e: feat[a:e], q_h,
                                qc.reshape(16, -1, w.ma), w.n_shapes, "gaussian", w.sigma)
    st = rel_err_stats(got, ref)
    record_parity("c4", "fif_scores_gaussian_vs_oracle_16q_x_1M", st)
    assert st["max"] <= RTOL and st["zero_mismatch"] == 0
    # (3) 8 DB shapes' self-join rows (index.py:196-210: the full view matrix)
    rows8 = samp[:8]
    Q8 = samp_views[:8]
    qc8 = scale.quantize_many_mt(C, Q8.reshape(-1, w.dim), w.ma).reshape(8, -1, w.ma)
    qc8 = np.where(Q8.any(axis=2)[:, :, None], qc8, -1)
    S8 = scale.fif_scores_many(cell_off, post_ord, lambda a, e: feat[a:e], Q8, qc8,
                               w.n_shapes, "gaussian", w.sigma)
    acts8, _ = scale.activations_from_scores(S8, w.k1, w.k2)
    ri, rv, rc = _raw_arrays(b)
    swaps = assert_topk_rows_close([(ri[j, :rc[j]], rv[j, :rc[j]]) for j in rows8],
                                   [(a.idx, a.val) for a in acts8])
    record_parity("c4", "self_join_raw_activations_8_shapes", {"raw_swaps": swaps})
    # (4) S-IF and rankings
    _check_scale_rerank("c4", b, w, ref, q, ids)


def test_c3_sampled_queries_against_oracle():
    """Config 3 at full size: 100k shapes x 64 views x d=4096 f32 (105 GB),
    K=1024, ma=2, streamed build (the index keeps only the tensor-core
    planes).  The database is regenerated block by block for the oracle: the
    16 queries scored against all 100k shapes, sampled DB views' assignments
    bit-exact, the list sizes per cell, 4 DB shapes' self-join rows, the
    S-IF and the rankings."""
    w = synth.WORKLOADS["c3"]
    mix = synth.BlockMixture(w, SEED, dev())
    C = synth.sample_centroids_rows(mix, w.K, SEED + 1).cpu().numpy()
    cbk = Codebook(C)
    ids = synth.shape_ids(w.n_shapes)
    cfg = gift.IndexConfig(n_views=w.n_views, codebook_size=w.K, ma=w.ma, k1=w.k1, k2=w.k2,
                           similarity="gaussian", sigma=w.sigma, batch_size=w.batch,
                           imported=True)
    b = gift.build_index_streamed(mix.provider(), ids, w.n_views, w.dim, cfg,
                                  codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")},
                                  chunk=1024, keep_features=False, self_join_batch=w.batch)
    f = b.fifs["A"].dev
    cell_off = f.cell_off.cpu().numpy()
    rng = np.random.default_rng(3)
    qs = mix.queries()
    sel = np.sort(rng.choice(qs.shape[0], 16, replace=False))
    q = qs[torch.from_numpy(sel).to(dev())].contiguous()
    q_h = q.cpu().numpy()
    qc = scale.quantize_many_mt(C, q_h.reshape(-1, w.dim), w.ma)
    np.testing.assert_array_equal(quantize_batch(cbk, q.reshape(-1, w.dim), w.ma), qc)
    qc = qc.reshape(16, w.n_views, w.ma)
    self_rows = np.sort(rng.choice(w.n_shapes, 4, replace=False))
    q4 = np.concatenate([mix.rows(int(r), int(r) + 1).cpu().numpy() for r in self_rows])
    qc4 = scale.quantize_many_mt(C, q4.reshape(-1, w.dim), w.ma).reshape(4, w.n_views, w.ma)
    qall = np.concatenate([q_h, q4])  # the 16 queries and 4 DB shapes' self-join rows
    qcall = np.concatenate([qc, qc4])
    best = np.zeros((20, w.n_views, w.n_shapes))
    sizes = np.zeros(w.K, dtype=np.int64)
    blk = 2048
    for s0 in range(0, w.n_shapes, blk):  # regenerate, assign (GPU), score (host)
        s1 = min(w.n_shapes, s0 + blk)
        X = mix.rows(s0, s1)
        flat = X.reshape(-1, w.dim)
        cells = quantize_batch(cbk, flat, 1)[:, 0].reshape(s1 - s0, w.n_views)
        Xh = X.cpu().numpy()
        if s0 == 0:  # the device assignments of a sample of views, bit-exact
            pick = rng.choice(flat.shape[0], 2048, replace=False)
            np.testing.assert_array_equal(
                scale.quantize_many_mt(C, Xh.reshape(-1, w.dim)[pick], 1)[:, 0],
                cells.reshape(-1)[pick])
        co, po, rows = scale.fif_lists(Xh, cells, w.K)
        sizes += np.diff(co)
        fr = Xh.reshape(-1, w.dim)
        best[:, :, s0:s1] = scale.fif_scores_many(co, po + s0, lambda a, e: fr[rows[a:e]], qall,
                                                  qcall, s1 - s0, "gaussian", w.sigma,
                                                  shape_base=s0, return_best=True)
        del X, Xh, fr
    np.testing.assert_array_equal(np.diff(cell_off), sizes)  # every cell's size
    ref = best[:16].sum(axis=1) / w.n_views
    got = mt.query_fif_batch(b.fifs["A"], q, w.ma, "gaussian", w.sigma).cpu().numpy()
    st = rel_err_stats(got, ref)
    record_parity("c3", "fif_scores_gaussian_vs_oracle_16q_x_100k", st)
    assert st["max"] <= RTOL and st["zero_mismatch"] == 0
    best4 = best[16:]
    acts4, _ = scale.activations_from_scores(best4.sum(axis=1) / w.n_views, w.k1, w.k2)
    ri, rv, rc = _raw_arrays(b)
    swaps = assert_topk_rows_close([(ri[j, :rc[j]], rv[j, :rc[j]]) for j in self_rows],
                                   [(a.idx, a.val) for a in acts4])
    record_parity("c3", "self_join_raw_activations_4_shapes", {"raw_swaps": swaps})
    _check_scale_rerank("c3", b, w, ref, q, ids)
