"""Index persistence: the bundle directory written by
the reference's `save_bundle` (index.py:360-375; codebook.py:127-145,
matching.py:164-211, rerank.py:233-323) against this package's writer and
reader.  Golden files: tests/golden/bundle_{tiny,small}.npz, the reference's
own bytes (make_golden.py `golden_bundles`)."""

import os
import tempfile

import numpy as np
import pytest

from cases import E2E_CASES, mixture_views, shape_ids
from conftest import load_golden
from helpers import RTOL, assert_ranking_close

CASES = E2E_CASES[:2]
BYTE_EXACT = ("config.json", "shapes.tsv", "codebook_A.bin", "codebook_B.bin",
              "fif_A.bin", "fif_B.bin")


def ref_files(name):
    g = load_golden(f"bundle_{name}.npz")
    return {k[len("file:"):]: g[k].tobytes() for k in g}


def write_dir(files, root):
    os.makedirs(root, exist_ok=True)
    for fn, data in files.items():
        with open(os.path.join(root, fn), "wb") as fh:
            fh.write(data)
    return root


# ------------------------------------------------------------------ host side (CPU)
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_host_formats_round_trip_reference_bytes(case):
    """Codebook and activation files: read the reference's bytes, write them
    back with this package's writers, get the same bytes."""
    from paper_1604_01879_b200 import codebook as cb
    from paper_1604_01879_b200 import rerank as rr

    files = ref_files(case[0])
    assert set(files) == set(BYTE_EXACT) | {"activations_A.bin", "activations_B.bin", "sif.bin"}
    with tempfile.TemporaryDirectory() as td:
        src = write_dir(files, os.path.join(td, "ref"))
        for ch in ("A", "B"):
            c = cb.load_codebook(os.path.join(src, f"codebook_{ch}.bin"))
            assert c.channel == ch and c.k == case[6]
            cb.save_codebook(c, os.path.join(td, "cb.bin"))
            assert open(os.path.join(td, "cb.bin"), "rb").read() == files[f"codebook_{ch}.bin"]
            acts = rr.load_activations(os.path.join(src, f"activations_{ch}.bin"))
            assert [a.owner for a in acts] == shape_ids(case[2])
            rr.save_activations(acts, os.path.join(td, "act.bin"))
            assert open(os.path.join(td, "act.bin"), "rb").read() == \
                files[f"activations_{ch}.bin"]


def test_truncated_files_raise_format_error():
    from paper_1604_01879_b200 import codebook as cb
    from paper_1604_01879_b200 import rerank as rr
    from paper_1604_01879_b200.errors import FormatError

    files = ref_files("tiny")
    with tempfile.TemporaryDirectory() as td:
        for fn, loader in (("codebook_A.bin", cb.load_codebook),
                           ("activations_A.bin", rr.load_activations)):
            p = os.path.join(td, fn)
            with open(p, "wb") as fh:
                fh.write(files[fn][: len(files[fn]) // 2])
            with pytest.raises(FormatError):
                loader(p)


# ------------------------------------------------------------------ device side (GPU)
def _gpu_bundle(case):
    from test_gpu_parity import _e2e_bundle

    return _e2e_bundle(case)


def _parse_acts(data, tmp):
    from paper_1604_01879_b200 import rerank as rr

    p = os.path.join(tmp, "x.bin")
    with open(p, "wb") as fh:
        fh.write(data)
    return rr.load_activations(p)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_gpu_built_bundle_saves_reference_bytes(case):
    """A bundle built on the GPU saves config/shapes/codebooks/F-IF lists
    byte-identical to the reference's; activation and S-IF files carry the
    identical supports with values within the score tolerance."""
    import paper_1604_01879_b200 as gift
    from paper_1604_01879_b200 import rerank as rr

    files = ref_files(case[0])
    bundle = _gpu_bundle(case)[0]
    with tempfile.TemporaryDirectory() as td:
        out = gift.save_bundle(bundle, os.path.join(td, "gpu"))
        got = {fn: open(os.path.join(out, fn), "rb").read() for fn in os.listdir(out)}
        assert set(got) == set(files)
        for fn in BYTE_EXACT:
            assert got[fn] == files[fn], fn
        for ch in ("A", "B"):
            a = _parse_acts(got[f"activations_{ch}.bin"], td)
            r = _parse_acts(files[f"activations_{ch}.bin"], td)
            for x, y in zip(a, r, strict=True):
                assert x.owner == y.owner
                np.testing.assert_array_equal(x.indices, y.indices)
                np.testing.assert_allclose(x.values, y.values, rtol=RTOL, atol=1e-12)
        sg = rr.load_sif(write_dir({"sif.bin": got["sif.bin"]}, os.path.join(td, "s1")) +
                         "/sif.bin")
        sr = rr.load_sif(write_dir({"sif.bin": files["sif.bin"]}, os.path.join(td, "s2")) +
                         "/sif.bin")
        assert sg.shape_ids == sr.shape_ids
        np.testing.assert_allclose(sg.norms, sr.norms, rtol=RTOL)
        for o1, o2, v1, v2 in zip(sg.entry_ordinals, sr.entry_ordinals, sg.entry_values,
                                  sr.entry_values, strict=True):
            np.testing.assert_array_equal(o1, o2)
            np.testing.assert_allclose(v1, v2, rtol=RTOL, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_reference_bundle_loads_and_serves(case):
    """The reference's saved directory loads into the GPU engine and its
    queries / query_by_id rank like the reference (e2e goldens)."""
    import paper_1604_01879_b200 as gift
    from paper_1604_01879_b200.features import ViewSet

    name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv = case
    g = load_golden(f"e2e_{name}.npz")
    views, _ = mixture_views(seed, N, V, d, classes, zero_views=zv, n_queries=nq)
    qs = views[N:]
    ids = shape_ids(N)
    with tempfile.TemporaryDirectory() as td:
        bundle = gift.load_bundle(write_dir(ref_files(name), os.path.join(td, "ref")))
        assert bundle.shape_ids == ids and bundle.config.ma == ma
        for rerank, tag in ((True, "rr"), (False, "nr")):
            for qi, q in enumerate(qs):
                res, _ = gift.query(bundle, ViewSet.from_matrix("query", q), top_k=top_k,
                                    rerank=rerank)
                assert_ranking_close([ids.index(r[0]) for r in res], [r[1] for r in res],
                                     g[f"q_{tag}_ids"][qi], g[f"q_{tag}_scores"][qi])
            for j, i in enumerate(range(0, N, max(1, N // 8))):
                res, _ = gift.query_by_id(bundle, ids[i], top_k=top_k, rerank=rerank)
                assert_ranking_close([ids.index(r[0]) for r in res], [r[1] for r in res],
                                     g[f"id_{tag}_ids"][j], g[f"id_{tag}_scores"][j])
        # and the re-saved directory is the reference's, byte for byte
        out = gift.save_bundle(bundle, os.path.join(td, "again"))
        for fn in os.listdir(out):
            assert open(os.path.join(out, fn), "rb").read() == ref_files(name)[fn], fn


@pytest.mark.gpu
def test_build_index_trains_codebooks_like_the_reference():
    """build_index(manifest, feature_files) without codebooks: each channel's
    codebook is trained on the device (k-means++ / Lloyd, index.py:186-193)
    and the saved bundle equals the reference's build_index output
    (tests/golden/bundle_trained.npz): config, shapes, codebooks and F-IF
    lists byte for byte; activations and S-IF on the same supports within
    the score tolerance."""
    import paper_1604_01879_b200 as gift
    from paper_1604_01879_b200 import rerank as rr

    g = load_golden("bundle_trained.npz")
    files = {k[len("file:"):]: g[k].tobytes() for k in g if k.startswith("file:")}
    labels = list(g["labels"])
    ids = shape_ids(len(labels))
    with tempfile.TemporaryDirectory() as td:
        paths = {}
        for ch in ("A", "B"):
            paths[ch] = os.path.join(td, f"feat_{ch}.bin")
            with open(paths[ch], "wb") as fh:
                fh.write(g[f"feat_{ch}"].tobytes())
        rows = [(f"/meshes/{s}.off", lab) for s, lab in zip(ids, labels)]
        cfg = gift.IndexConfig(n_views=6, codebook_size=8, ma=2, k1=5, k2=2)
        bundle = gift.build_index(rows, cfg, feature_files=paths)
        out = gift.save_bundle(bundle, os.path.join(td, "gpu"))
        got = {fn: open(os.path.join(out, fn), "rb").read() for fn in os.listdir(out)}
        assert set(got) == set(files)
        for fn in BYTE_EXACT:
            assert got[fn] == files[fn], fn
        for ch in ("A", "B"):
            a = _parse_acts(got[f"activations_{ch}.bin"], td)
            r = _parse_acts(files[f"activations_{ch}.bin"], td)
            for x, y in zip(a, r, strict=True):
                assert x.owner == y.owner
                np.testing.assert_array_equal(x.indices, y.indices)
                np.testing.assert_allclose(x.values, y.values, rtol=RTOL, atol=1e-12)
        sg = rr.load_sif(write_dir({"sif.bin": got["sif.bin"]}, os.path.join(td, "s1")) +
                         "/sif.bin")
        sr = rr.load_sif(write_dir({"sif.bin": files["sif.bin"]}, os.path.join(td, "s2")) +
                         "/sif.bin")
        for o1, o2, v1, v2 in zip(sg.entry_ordinals, sr.entry_ordinals, sg.entry_values,
                                  sr.entry_values, strict=True):
            np.testing.assert_array_equal(o1, o2)
            np.testing.assert_allclose(v1, v2, rtol=RTOL, atol=1e-12)
