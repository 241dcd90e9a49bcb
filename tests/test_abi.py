"""The C-ABI library loads and exports every symbol include/gift.h declares
(no compute calls: CPU only)."""

import os
import re

import pytest

from conftest import ROOT


def header_functions():
    src = open(os.path.join(ROOT, "include", "gift.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gift_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    fns = header_functions()
    for must in ("gift_quantize", "gift_fif_gather", "gift_fif_segments", "gift_fif_tiles",
                 "gift_fif_score", "gift_topk_rows", "gift_act_mean", "gift_act_aggregate",
                 "gift_sif_query", "gift_radix_sort_pairs", "gift_last_error"):
        assert must in fns


def test_library_exports_every_header_symbol():
    from paper_1604_01879_b200 import _native

    lib = _native.load_library()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert set(header_functions()) == set(_native.EXPORTED)
    assert lib.gift_version() == 1
    assert lib.gift_fif_tile_n() == 128


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_1604_01879_b200", "libgift.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


def test_no_cpu_fallback_without_gpu():
    import torch

    from paper_1604_01879_b200 import _native, errors
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    _native._lib = None
    with pytest.raises(errors.NativeUnavailable):
        _native.lib()
