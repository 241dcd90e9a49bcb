"""ctypes binding of libgift.so (include/gift.h) and torch plumbing helpers.

The library is the product path: every numeric step of the GIFT query path
runs in its sm_100a kernels.  There is no CPU fallback — if the library or a
CUDA device is missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgift.so")

GIFT_F32, GIFT_F16, GIFT_F64 = 0, 1, 2
SIM_COSINE, SIM_GAUSSIAN = 0, 1
FIF_TILED_SEGMENTS = 1  # gift_fif_view.flags (include/gift.h)
# kernel variants selected through gift_fif_view.flags (include/gift.h)
FIF_SCAN_SIMT = 1 << 16
FIF_QUANT_SIMT = 1 << 17
FIF_REDUCE = {"auto": 0, "range": 1 << 18, "gather": 2 << 18, "owner": 3 << 18}
FIF_SCHED_STATIC = 1 << 20
FIF_PAIR = {"auto": 0, "off": 1 << 21, "on": 2 << 21}
FIF_RAW_ACCUM = 1 << 29
FIF_DENSE_OFF = 1 << 30
FIF_VARIANT_MASK = ((1 << 16) | (1 << 17) | (3 << 18) | (1 << 20) | (3 << 21) | (31 << 24)
                    | FIF_RAW_ACCUM | FIF_DENSE_OFF)
QUANT_SIMT = 1        # gift_quantize_ex flags
SIF_ROWS, SIF_SORT, SIF_BUCKET = 1, 2, 4  # gift_sif_query_topk flags


def fif_reserve_sms(n: int) -> int:
    """GIFT_FIF_RESERVE_SMS(n): flags bits 8-15."""
    return (int(n) & 255) << 8


def fif_drain_kb(n: int) -> int:
    """GIFT_FIF_DRAIN_KB(n): flags bits 24-28 (1..16; 0 = the library default, 8)."""
    return (int(n) & 31) << 24

_c_i32 = ctypes.c_int32
_c_i64 = ctypes.c_int64
_c_sz = ctypes.c_size_t
_c_dbl = ctypes.c_double
_c_p = ctypes.c_void_p


class FifView(ctypes.Structure):
    """Mirror of `gift_fif_view` (include/gift.h)."""
    _fields_ = [
        ("K", _c_i32), ("d", _c_i32), ("dtype", _c_i32), ("flags", _c_i32),
        ("n_postings", _c_i64), ("n_segments", _c_i64), ("n_tiles", _c_i64),
        ("n_local", _c_i64), ("ord_base", _c_i64),
        ("cell_off", _c_p), ("post_ord", _c_p), ("feat", _c_p), ("pnorm2", _c_p),
        ("seg_off", _c_p), ("seg_ord", _c_p), ("seg_pstart", _c_p),
        ("tile_off", _c_p), ("tile_pstart", _c_p), ("tile_pend", _c_p),
        ("tile_seg0", _c_p), ("tile_seg1", _c_p),
        ("centroids", _c_p), ("cnorm2", _c_p), ("cmax_norm", _c_dbl),
        ("feat_hi", _c_p), ("feat_lo", _c_p),
        ("shape_seg_off", _c_p), ("shape_seg", _c_p), ("shape_seg_cell", _c_p),
        ("max_cell_segments", _c_i64), ("seg_single", _c_p),
    ]


_SIGS = {
    "gift_version": (_c_i32, []),
    "gift_last_error": (_c_i32, [ctypes.c_char_p, _c_sz]),
    "gift_fif_tile_n": (_c_i32, []),
    "gift_quantize_ws_bytes": (_c_sz, [_c_i64, _c_i32, _c_i32, _c_i32]),
    "gift_quantize": (_c_i32, [_c_p, _c_i32, _c_i64, _c_i32, _c_p, _c_p, _c_i32, _c_dbl, _c_i32,
                               _c_p, _c_i32, _c_p, _c_p, _c_sz, _c_p]),
    "gift_quantize_ex": (_c_i32, [_c_p, _c_i32, _c_i64, _c_i32, _c_p, _c_p, _c_i32, _c_dbl,
                                  _c_i32, _c_p, _c_i32, _c_p, _c_p, _c_sz, _c_i32, _c_p]),
    "gift_rows_sqnorm_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_p, _c_p]),
    "gift_kmeans_assign": (_c_i32, [_c_p, _c_i64, _c_i32, _c_p, _c_i32, _c_p, _c_p, _c_p, _c_p,
                                    _c_p]),
    "gift_kmeans_update": (_c_i32, [_c_p, _c_i64, _c_i32, _c_p, _c_p, _c_i32, _c_p, _c_p]),
    "gift_normalize_rows": (_c_i32, [_c_p, _c_p, _c_i64, _c_i32, _c_p, _c_p]),
    "gift_view_prep": (_c_i32, [_c_p, _c_i32, _c_i64, _c_i32, _c_p, _c_p, _c_p]),
    "gift_radix_sort_ws_bytes": (_c_sz, [_c_i64]),
    "gift_radix_sort_pairs": (_c_i32, [_c_p, _c_p, _c_i64, _c_i32, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "gift_offsets_from_sorted": (_c_i32, [_c_p, _c_i64, _c_i64, _c_p, _c_p]),
    "gift_fif_gather": (_c_i32, [_c_p, _c_i32, _c_i32, _c_i32, _c_p, _c_i64, _c_i64, _c_p, _c_p,
                                 _c_p, _c_p]),
    "gift_perm_invert": (_c_i32, [_c_p, _c_i64, _c_i64, _c_p, _c_p]),
    "gift_fif_scatter": (_c_i32, [_c_p, _c_i32, _c_i32, _c_i32, _c_i64, _c_p, _c_i64, _c_i64, _c_p,
                                  _c_p, _c_p, _c_p, _c_p, _c_p]),
    "gift_fif_build_ws_bytes": (_c_sz, [_c_i64, _c_i32]),
    "gift_fif_segments": (_c_i32, [_c_p, _c_p, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_sz,
                                   _c_p]),
    "gift_fif_tiles": (_c_i32, [_c_p, _c_p, _c_p, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p,
                                _c_p, _c_sz, _c_p]),
    "gift_split_planes": (_c_i32, [_c_p, _c_i64, _c_p, _c_p, _c_p]),
    "gift_gather_rows_f32": (_c_i32, [_c_p, _c_i32, _c_i32, _c_p, _c_i64, _c_p, _c_p]),
    "gift_gather_rows_planes": (_c_i32, [_c_p, _c_p, _c_i32, _c_p, _c_i64, _c_p, _c_p]),
    "gift_fif_score_ws_bytes": (_c_sz, [ctypes.POINTER(FifView), _c_i32, _c_i32, _c_i32, _c_i64]),
    "gift_fif_score": (_c_i32, [ctypes.POINTER(FifView), _c_p, _c_i32, _c_i32, _c_p, _c_i32,
                                _c_i32, _c_dbl, _c_p, _c_p, _c_sz, _c_p]),
    "gift_fif_score_ex": (_c_i32, [ctypes.POINTER(FifView), _c_p, _c_i32, _c_i32, _c_p, _c_i32,
                                   _c_i32, _c_dbl, _c_p, _c_p, _c_sz, _c_p, _c_p, _c_p]),
    "gift_fif_score_ranges": (_c_i32, [ctypes.POINTER(FifView), _c_i32]),
    "gift_fif_score_ranges2": (_c_i32, [ctypes.POINTER(FifView), _c_i32, _c_i32]),
    "gift_fif_reduce_mode": (_c_i32, [ctypes.POINTER(FifView), _c_i32, _c_i32]),
    "gift_fif_score_ex2": (_c_i32, [ctypes.POINTER(FifView), _c_p, _c_i32, _c_i32, _c_p, _c_i32,
                                    _c_i32, _c_dbl, _c_p, _c_p, _c_sz, _c_p, _c_p, _c_p, _c_i32,
                                    _c_p, _c_p]),
    "gift_topk_cand": (_c_i32, [_c_p, _c_p, _c_i32, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p]),
    "gift_topk_cand_tb": (_c_i32, [_c_p, _c_p, _c_p, _c_i32, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                   _c_p]),
    "gift_topk_rows": (_c_i32, [_c_p, _c_i32, _c_i64, _c_i32, _c_p, _c_p, _c_i64, _c_i32, _c_p,
                                _c_p, _c_p]),
    "gift_topk_ws_bytes": (_c_sz, [_c_i32, _c_i64, _c_i32]),
    "gift_topk_rows_ex": (_c_i32, [_c_p, _c_i32, _c_i64, _c_i32, _c_p, _c_p, _c_i64, _c_i32, _c_p,
                                   _c_p, _c_p, _c_sz, _c_p]),
    "gift_act_from_topk": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_p,
                                    _c_p, _c_p]),
    "gift_act_mean": (_c_i32, [_c_p, _c_p, _c_p, _c_i32, _c_p, _c_i32, _c_i32, _c_i32, _c_p, _c_p,
                               _c_p, _c_p, _c_p]),
    "gift_act_aggregate": (_c_i32, [_c_p, _c_p, _c_p, _c_i32, _c_p, _c_p, _c_p, _c_i32, _c_i32,
                                    _c_dbl, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "gift_act_compact": (_c_i32, [_c_p, _c_p, _c_p, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                                  _c_p, _c_sz, _c_p]),
    "gift_sif_permute": (_c_i32, [_c_p, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_p]),
    "gift_sif_query": (_c_i32, [_c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p,
                                _c_i32, _c_i32, _c_p, _c_p]),
    "gift_sif_query_topk_ws_bytes": (_c_sz, [_c_i32, _c_i32, _c_i64, _c_i32, _c_i64, _c_i32]),
    "gift_sif_query_topk": (_c_i32, [_c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p,
                                     _c_p, _c_i32, _c_i32, _c_p, _c_i32, _c_i64, _c_p, _c_p, _c_p,
                                     _c_i64, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_sz, _c_i32,
                                     _c_p]),
    "gift_exact_sets": (_c_i32, [_c_p, _c_i32, _c_p, _c_i32, _c_i32, _c_p, _c_i32, _c_p, _c_i32,
                                 _c_i32, _c_i32, _c_p, _c_p]),
    "gift_eval_ranks": (_c_i32, [_c_p, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_i32, _c_p, _c_p]),
    "gift_fif_score_f64_ws_bytes": (_c_sz, [_c_i32, _c_i32, _c_i64]),
    "gift_fif_score_f64": (_c_i32, [_c_p, _c_i32, _c_i32, _c_i32, _c_p, _c_i32, _c_i32, _c_p,
                                    _c_p, _c_p, _c_i64, _c_i64, _c_i32, _c_dbl, _c_p, _c_sz,
                                    _c_p, _c_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libgift.so and bind every entry point (no GPU needed)."""
    if not os.path.exists(path):
        raise errors.NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib() -> ctypes.CDLL:
    """The loaded library; requires a CUDA device (no CPU fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not torch.cuda.is_available():
                    raise errors.NativeUnavailable(
                        "no CUDA device: the GIFT path runs only on the sm_100a kernels")
                _lib = load_library()
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    lib().gift_last_error(buf, 1024)
    return buf.value.decode("utf-8", "replace")


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    raise errors.from_status(rc, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def ptr(t) -> int | None:
    """Device (or host) address of a tensor, None for None."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def device() -> torch.device:
    lib()
    return torch.device("cuda", torch.cuda.current_device())


class Workspace:
    """Grow-only per-stream scratch buffer (caller-owned memory for the ABI)."""

    def __init__(self):
        self._buf = None
        self._captured = False  # a CUDA graph (GraphedQuery) addresses the buffer
        self._retired = []

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if torch.cuda.is_current_stream_capturing():
            self._captured = True
        if self._buf is None or self._buf.numel() < nbytes:
            if self._buf is not None and self._captured:
                self._retired.append(self._buf)  # the graph's kernels still use it
            self._buf = None
            self._buf = torch.empty(nbytes, dtype=torch.uint8, device=device())
        return self._buf


_ws_local = threading.local()


def workspace(slot: str = "default", stream=None) -> Workspace:
    """Scratch buffer of `slot` for the launches on `stream` (default: the
    current stream): work queued on different streams never shares scratch."""
    d = getattr(_ws_local, "pool", None)
    if d is None:
        d = _ws_local.pool = {}
    key = (slot, stream_ptr(stream))
    ws = d.get(key)
    if ws is None:
        ws = d[key] = Workspace()
    return ws
