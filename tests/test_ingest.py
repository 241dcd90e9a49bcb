"""Feature ingest: GIFTFT1 files streamed to the
device and re-normalized there, bit-identical to the reference's
import_features (features.py:67-71, :140-185).  Golden: tests/golden/
ingest.npz -- a file written by the reference's write_features and the
reference's import_features result on it (make_golden.py `golden_ingest`)."""

import os
import struct
import tempfile

import numpy as np
import pytest

from conftest import load_golden


def _golden_file(td):
    g = load_golden("ingest.npz")
    p = os.path.join(td, "feat.bin")
    with open(p, "wb") as fh:
        fh.write(g["blob"].tobytes())
    return p, g


def _normalize_host(raw, norms):
    """features.py:67-71 given the norms: f32(row_f64 / norm), zero-norm rows
    unchanged -- the arithmetic gift_normalize_rows performs on the device."""
    m = raw.reshape(-1, raw.shape[-1]).astype(np.float64)
    nr = norms[:, None]
    safe = np.where(nr == 0.0, 1.0, nr)
    out = np.where(nr == 0.0, m, m / safe).astype(np.float32)
    return out.reshape(raw.shape)


# ------------------------------------------------------------------ host side (CPU)
def test_feature_file_parses_like_import_features():
    from paper_1604_01879_b200 import features as ft

    with tempfile.TemporaryDirectory() as td:
        p, g = _golden_file(td)
        f = ft.FeatureFile(p, "A")
        assert f.shape_ids == list(g["ids"])  # first position, last rows for the repeated id
        assert (f.n_views, f.dim) == g["mats"].shape[1:]
        raw = f.host_rows(range(len(f)))
        got = _normalize_host(raw, f.row_norms(raw))
        np.testing.assert_array_equal(got.view(np.uint32), g["mats"].view(np.uint32))
        # and the package's host import_features restatement agrees
        imp = ft.import_features(p, "A")
        assert list(imp) == list(g["ids"])
        for i, s in enumerate(imp):
            np.testing.assert_array_equal(imp[s].matrix("A").view(np.uint32),
                                          g["mats"][i].view(np.uint32))


def test_feature_file_errors():
    from paper_1604_01879_b200 import features as ft
    from paper_1604_01879_b200.errors import DimensionMismatch, FormatError

    with tempfile.TemporaryDirectory() as td:
        p, g = _golden_file(td)
        blob = open(p, "rb").read()
        for cut in (0, 5, 10, 13, 30, len(blob) // 2, len(blob) - 1):
            q = os.path.join(td, f"cut{cut}.bin")
            with open(q, "wb") as fh:
                fh.write(blob[:cut])
            with pytest.raises(FormatError):
                ft.FeatureFile(q)
            with pytest.raises(FormatError):
                ft.import_features(q, "A")
        q = os.path.join(td, "magic.bin")
        with open(q, "wb") as fh:
            fh.write(b"GIFTFT2\x00" + blob[8:])
        with pytest.raises(FormatError):
            ft.FeatureFile(q)
        # ragged view counts
        q = os.path.join(td, "ragged.bin")
        with open(q, "wb") as fh:
            fh.write(ft.FEATURE_MAGIC + struct.pack("<I", 2))
            for sid, nv in (("x", 2), ("y", 3)):
                fh.write(struct.pack("<H", 1) + sid.encode() + struct.pack("<II", nv, 4))
                fh.write(np.ones((nv, 4), dtype="<f4").tobytes())
        with pytest.raises(DimensionMismatch):
            ft.FeatureFile(q)
        # an empty shape list parses to nothing
        q = os.path.join(td, "empty.bin")
        with open(q, "wb") as fh:
            fh.write(ft.FEATURE_MAGIC + struct.pack("<I", 0))
        assert len(ft.FeatureFile(q)) == 0


def test_write_features_reproduces_reference_bytes():
    """The package's writer, fed the parsed raw rows of the unique ids in
    file order, writes the reference writer's bytes (ids repeated in the
    golden file are written once here, so compare against a re-parse)."""
    from paper_1604_01879_b200 import features as ft

    with tempfile.TemporaryDirectory() as td:
        p, g = _golden_file(td)
        f = ft.FeatureFile(p, "A")
        raw = f.host_rows(range(len(f)))
        vss = [ft.ViewSet.from_matrix(s, raw[i], channels=("A",)) for i, s in enumerate(f.shape_ids)]
        q = os.path.join(td, "again.bin")
        ft.write_features(q, vss, "A")
        f2 = ft.FeatureFile(q, "A")
        assert f2.shape_ids == f.shape_ids
        np.testing.assert_array_equal(f2.host_rows(range(len(f2))), raw)


# ------------------------------------------------------------------ device side (GPU)
@pytest.mark.gpu
@pytest.mark.parametrize("chunk_bytes", [1 << 30, 6 * 300 * 4 * 2])
def test_device_ingest_bit_identical_to_reference(chunk_bytes):
    from paper_1604_01879_b200 import features as ft

    with tempfile.TemporaryDirectory() as td:
        p, g = _golden_file(td)
        f = ft.FeatureFile(p, "A")
        sel = [4, 0, 2, 2, 1, 3]  # any order, repeats allowed
        x = f.device_rows(sel, chunk_bytes=chunk_bytes).cpu().numpy()
        np.testing.assert_array_equal(x.view(np.uint32), g["mats"][sel].view(np.uint32))


@pytest.mark.gpu
def test_build_index_from_feature_files_matches_host_import():
    """build_index(manifest, feature_files=...) through the device ingest
    ranks exactly like an index built from the host import_features rows."""
    import paper_1604_01879_b200 as gift
    from cases import mixture_views, shape_ids
    from paper_1604_01879_b200 import features as ft
    from paper_1604_01879_b200.codebook import Codebook

    views, _ = mixture_views(31, 60, 6, 32, 5, n_queries=4)
    raw = views * np.float32(3.0)  # not unit norm: the ingest must re-normalize
    ids = shape_ids(60)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "f.bin")
        ft.write_features(p, [ft.ViewSet.from_matrix(s, raw[i], channels=("A",))
                              for i, s in enumerate(ids)], "A")
        man = [(os.path.join(td, s + ".off"), "c") for s in ids[::-1]]  # manifest order rules
        imp = ft.import_features(p, "A")
        host = np.stack([imp[s].matrix("A") for s in ids[::-1]])
        C = host.reshape(-1, 32)[::7][:8].copy()
        cfg = gift.IndexConfig(n_views=6, codebook_size=8, ma=2, k1=5, k2=2)
        cbs = {"A": Codebook(C, "A"), "B": Codebook(C, "B")}
        b1 = gift.build_index(man, cfg, feature_files={"A": p, "B": p}, codebooks=cbs)
        b2 = gift.build_index_from_views(host, ids[::-1], cfg, codebooks=cbs,
                                         labels={s: "c" for s in ids})
        assert b1.shape_ids == b2.shape_ids
        for q in views[60:]:
            r1, _ = gift.query(b1, ft.ViewSet.from_matrix("q", q), top_k=20)
            r2, _ = gift.query(b2, ft.ViewSet.from_matrix("q", q), top_k=20)
            assert [x[:2] for x in r1] == [x[:2] for x in r2]
        b3 = gift.build_index_from_feature_file(p, cfg, codebooks=cbs, chunk=16,
                                                self_join_batch=16)
        assert b3.shape_ids == ids
