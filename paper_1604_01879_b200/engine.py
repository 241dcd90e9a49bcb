"""Device engine: host orchestration of the libgift kernels.

All tensors here live on the GPU; every numeric step is a libgift kernel
(the ABI of include/gift.h).  PyTorch provides allocation, streams and the
odd reshape/copy (plumbing only).  Layouts in HBM:

  DeviceFif   cell-major CSR of one shard: cell_off[K+1] i64, post_ord[P] i32
              (global ordinal), feat[P, d] f32|f16, pnorm2[P] f32, the
              (cell, shape) segments seg_off[K+1]/seg_ord[S]/seg_pstart[S+1],
              scan tiles tile_*[T], and the shape -> postings map
              shape_off[n_local+1]/shape_post[P] (query_by_id).
  ActRows     fixed-capacity activation rows: idx[n, cap] i32 ascending,
              val[n, cap] f64, cnt[n] i32, norm[n] f64.
  DeviceSif   CSR over the global coordinate i: e_off[N+1] i64,
              e_ord[nnz] i32 (local owner), e_val[nnz] f64, norms[n_local].
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .errors import DimensionMismatch, EmptySet, Unsupported

_DTYPE_CODE = {torch.float32: nat.GIFT_F32, torch.float16: nat.GIFT_F16,
               torch.float64: nat.GIFT_F64}




def _bits(n: int) -> int:
    return max(1, int(n).bit_length())


def _sp(stream=None):
    return nat.stream_ptr(stream)


# ------------------------------------------------------------------ codebook
@dataclass
class DeviceCodebook:
    centroids: torch.Tensor  # [K, d] f32
    cnorm2: torch.Tensor     # [K] f64
    cmax: float

    @property
    def K(self) -> int:
        return self.centroids.shape[0]

    @property
    def d(self) -> int:
        return self.centroids.shape[1]

    @classmethod
    def from_numpy(cls, centroids: np.ndarray) -> "DeviceCodebook":
        c = np.ascontiguousarray(centroids, dtype=np.float32)
        c64 = c.astype(np.float64)
        n2 = (c64 * c64).sum(axis=1)
        dev = nat.device()
        return cls(torch.from_numpy(c).to(dev), torch.from_numpy(n2).to(dev),
                   float(np.sqrt(n2.max())) if len(n2) else 0.0)


def quantize_rows(cb: DeviceCodebook, X: torch.Tensor, ma: int, nz: torch.Tensor | None = None,
                  zero_key: int = -1, stream=None, flags: int = 0) -> torch.Tensor:
    """K1: [n, d] (f32/f16/f64, device) -> [n, ma] int32 nearest centroids.
    flags: nat.QUANT_SIMT selects the CUDA-core stage 1 (same results)."""
    X = X.contiguous()
    n, d = X.shape
    if d != cb.d:
        raise DimensionMismatch(f"vector dim {d} != codebook dim {cb.d}")
    if not 1 <= ma <= cb.K:
        raise ValueError(f"ma must be in [1, {cb.K}]")
    out = torch.empty((n, ma), dtype=torch.int32, device=X.device)
    wsb = nat.lib().gift_quantize_ws_bytes(n, d, cb.K, _DTYPE_CODE[X.dtype])
    ws = nat.workspace("quantize", stream).get(wsb)
    nat.call("gift_quantize_ex", nat.ptr(X), _DTYPE_CODE[X.dtype], n, d, nat.ptr(cb.centroids),
             nat.ptr(cb.cnorm2), cb.K, cb.cmax, ma, nat.ptr(nz), zero_key, nat.ptr(out),
             nat.ptr(ws), ws.numel(), int(flags), _sp(stream))
    return out


def view_prep(X: torch.Tensor, stream=None):
    X = X.contiguous()
    n, d = X.shape
    nz = torch.empty(n, dtype=torch.uint8, device=X.device)
    n2 = torch.empty(n, dtype=torch.float32, device=X.device)
    nat.call("gift_view_prep", nat.ptr(X), _DTYPE_CODE[X.dtype], n, d, nat.ptr(nz), nat.ptr(n2),
             _sp(stream))
    return nz, n2


def radix_sort_pairs(keys: torch.Tensor, vals: torch.Tensor, key_bits: int, stream=None):
    """Stable sort of uint32 (as int32 storage) key/value pairs, in place."""
    n = keys.numel()
    if n <= 1:
        return keys, vals
    kt = torch.empty_like(keys)
    vt = torch.empty_like(vals)
    ws = nat.workspace("radix", stream).get(nat.lib().gift_radix_sort_ws_bytes(n))
    nat.call("gift_radix_sort_pairs", nat.ptr(keys), nat.ptr(vals), n, key_bits, nat.ptr(kt),
             nat.ptr(vt), nat.ptr(ws), ws.numel(), _sp(stream))
    return keys, vals


def offsets_from_sorted(keys: torch.Tensor, nbuckets: int, stream=None) -> torch.Tensor:
    off = torch.empty(nbuckets + 1, dtype=torch.int64, device=keys.device)
    nat.call("gift_offsets_from_sorted", nat.ptr(keys), keys.numel(), nbuckets, nat.ptr(off),
             _sp(stream))
    return off


# ------------------------------------------------------------------ F-IF
class DeviceFif:
    """One shard of the first inverted file (matching.py:64-133 semantics)."""

    def __init__(self):
        self.view = None
        self.feat = None
        self.feat_hi = self.feat_lo = None
        self.variant = 0  # kernel-variant bits of gift_fif_view.flags (set_variant)

    def set_variant(self, scan: str = "tc", quant: str = "tc", reduce: str = "auto",
                    pair: str = "auto", sched: str = "dynamic", drain_kb: int = 0,
                    raw_accum: bool = False, dense: str = "auto"):
        """Select kernel variants through the view flags (include/gift.h):
        scan/quant "tc" | "simt", reduce "auto" | "range" | "gather" | "owner",
        pair "auto" | "on" | "off", sched "dynamic" | "static", drain_kb 0..16
        (0 = default), raw_accum (no truncation compensation; measurement
        only), dense "auto" | "off" (fp16 storage: the probe-major pair scan
        of the cells with >= 192 probes per batch).  Defaults reproduce the
        measured-fastest choice."""
        v = (nat.FIF_SCAN_SIMT if scan == "simt" else 0) | \
            (nat.FIF_QUANT_SIMT if quant == "simt" else 0) | nat.FIF_REDUCE[reduce] | \
            nat.FIF_PAIR[pair] | (nat.FIF_SCHED_STATIC if sched == "static" else 0) | \
            nat.fif_drain_kb(drain_kb) | (nat.FIF_RAW_ACCUM if raw_accum else 0) | \
            (nat.FIF_DENSE_OFF if dense == "off" else 0)
        self.variant = v
        self.bind()
        return self

    @property
    def storage_dtype(self):
        """Storage dtype of the database features (f32 or f16); an index
        built without its storage copy keeps f32 semantics in the planes."""
        if self.feat is not None:
            return self.feat.dtype
        return torch.float32

    @property
    def device(self):
        return self.post_ord.device

    @property
    def P(self) -> int:
        return int(self.post_ord.numel())

    def bind(self):
        v = nat.FifView()
        v.K, v.d = self.cb.K, self.cb.d
        v.dtype = _DTYPE_CODE[self.storage_dtype]
        v.n_postings, v.n_segments, v.n_tiles = self.P, self.S, self.T
        v.n_local, v.ord_base = self.n_local, self.ord_base
        v.feat = None if self.feat is None else self.feat.data_ptr()
        for name in ("cell_off", "post_ord", "pnorm2", "seg_off", "seg_ord", "seg_pstart",
                     "tile_off", "tile_pstart", "tile_pend", "tile_seg0", "tile_seg1"):
            setattr(v, name, getattr(self, name).data_ptr())
        v.centroids = self.cb.centroids.data_ptr()
        v.cnorm2 = self.cb.cnorm2.data_ptr()
        v.cmax_norm = self.cb.cmax
        v.feat_hi = None if self.feat_hi is None else self.feat_hi.data_ptr()
        v.feat_lo = None if self.feat_lo is None else self.feat_lo.data_ptr()
        v.shape_seg_off = self.shape_seg_off.data_ptr()
        v.shape_seg = self.shape_seg.data_ptr()
        v.shape_seg_cell = self.shape_seg_cell.data_ptr()
        v.max_cell_segments = self.smax
        v.seg_single = self.seg_single.data_ptr()
        v.flags = (nat.FIF_TILED_SEGMENTS if self.seg_len_max <= nat.lib().gift_fif_tile_n()
                   else 0) | self.variant
        self.view = v
        return v

    @classmethod
    def build(cls, X: torch.Tensor, cb: DeviceCodebook, ord_base: int = 0, stream=None,
              assign: torch.Tensor | None = None) -> "DeviceFif":
        """K2: X = [n_local, V, d] f32|f16 device views of this shard's shapes
        (zero rows = empty views).  Postings are appended per cell in
        shape-major / view-minor order (matching.py:112-125)."""
        if X.dim() != 3:
            raise ValueError("views must be [n_shapes, n_views, d]")
        n_local, V, d = X.shape
        if d != cb.d:
            raise DimensionMismatch(f"view dim {d} != codebook dim {cb.d}")
        if X.dtype not in (torch.float32, torch.float16):
            raise ValueError("feature storage must be float32 or float16")
        dev = X.device
        X = X.contiguous()
        flat = X.view(n_local * V, d)
        K = cb.K
        self = cls()
        self.cb, self.ord_base, self.n_local, self.V, self.d = cb, int(ord_base), n_local, V, d
        nviews = n_local * V
        nz, _ = view_prep(flat, stream)
        if assign is None:
            keys = quantize_rows(cb, flat, 1, nz=nz, zero_key=K, stream=stream).view(-1)
        else:
            keys = torch.where(nz.bool(), assign.view(-1).to(torch.int32),
                               torch.full_like(assign.view(-1), K, dtype=torch.int32))
        keys = keys.contiguous()
        vals = torch.arange(nviews, dtype=torch.int32, device=dev)
        radix_sort_pairs(keys, vals, _bits(K), stream)
        cell_off_full = offsets_from_sorted(keys, K + 1, stream)  # [K+2]
        P = int(cell_off_full[K].item())
        self.cell_off = cell_off_full[: K + 1].contiguous()
        self.feat = torch.empty((P, d), dtype=X.dtype, device=dev)
        self.post_ord = torch.empty(P, dtype=torch.int32, device=dev)
        self.pnorm2 = torch.empty(P, dtype=torch.float32, device=dev)
        perm = vals[:P].contiguous()
        nat.call("gift_fif_gather", nat.ptr(flat), _DTYPE_CODE[X.dtype], d, V, nat.ptr(perm), P,
                 self.ord_base, nat.ptr(self.feat), nat.ptr(self.post_ord), nat.ptr(self.pnorm2),
                 _sp(stream))
        del keys, vals, perm
        self._finish(stream)
        return self

    @classmethod
    def build_streamed(cls, provider, n_local: int, V: int, d: int, cb: DeviceCodebook,
                       dtype=torch.float32, ord_base: int = 0, chunk: int = 512,
                       keep_features: bool = False, stream=None) -> "DeviceFif":
        """K2 over a database streamed in chunks of shapes (configs whose
        features do not fit HBM twice, e.g. config 3's 105 GB):
        `provider(s0, s1)` returns the device views [s1 - s0, V, d] of local
        shapes s0..s1 (f32 or the storage dtype).  Pass 1 quantizes every
        chunk into one key per view; the stable radix sort gives the same
        cell-major (ordinal, view) order as `build`; pass 2 re-reads the
        chunks and scatters their rows straight into the tensor-core planes
        (and the storage-dtype copy only with keep_features)."""
        if cb.d != d:
            raise DimensionMismatch(f"view dim {d} != codebook dim {cb.d}")
        if dtype not in (torch.float32, torch.float16):
            raise ValueError("feature storage must be float32 or float16")
        dev = cb.centroids.device
        K = cb.K
        self = cls()
        self.cb, self.ord_base, self.n_local, self.V, self.d = cb, int(ord_base), n_local, V, d
        nviews = n_local * V
        keys = torch.empty(nviews, dtype=torch.int32, device=dev)
        for s0 in range(0, n_local, chunk):
            s1 = min(n_local, s0 + chunk)
            X = provider(s0, s1).to(dtype).contiguous().view(-1, d)
            nz, _ = view_prep(X, stream)
            keys[s0 * V:s1 * V] = quantize_rows(cb, X, 1, nz=nz, zero_key=K,
                                                stream=stream).view(-1)
            del X
        vals = torch.arange(nviews, dtype=torch.int32, device=dev)
        radix_sort_pairs(keys, vals, _bits(K), stream)
        cell_off_full = offsets_from_sorted(keys, K + 1, stream)
        P = int(cell_off_full[K].item())
        self.cell_off = cell_off_full[: K + 1].contiguous()
        del keys
        pos = torch.empty(max(nviews, 1), dtype=torch.int32, device=dev)
        nat.call("gift_perm_invert", nat.ptr(vals), P, nviews, nat.ptr(pos), _sp(stream))
        del vals
        half = dtype == torch.float16
        tc = P > 0 and d % 8 == 0
        if not tc and not keep_features:
            raise ValueError("dropping the storage copy needs the tensor-core planes (d % 8 == 0)")
        self.feat = torch.empty((P, d), dtype=dtype, device=dev) if (keep_features or half) else None
        if half:
            self.feat_hi, self.feat_lo = self.feat, None
        elif tc:
            self.feat_hi = torch.empty((P, d), dtype=torch.float16, device=dev)
            self.feat_lo = torch.empty((P, d), dtype=torch.float16, device=dev)
        else:
            self.feat_hi = self.feat_lo = None
        self.post_ord = torch.empty(P, dtype=torch.int32, device=dev)
        self.pnorm2 = torch.empty(P, dtype=torch.float32, device=dev)
        for s0 in range(0, n_local, chunk):
            s1 = min(n_local, s0 + chunk)
            X = provider(s0, s1).to(dtype).contiguous()
            nat.call("gift_fif_scatter", nat.ptr(X), _DTYPE_CODE[dtype], d, V, (s1 - s0) * V,
                     nat.ptr(pos), s0 * V, self.ord_base,
                     None if half else nat.ptr(self.feat), nat.ptr(self.feat_hi),
                     None if half else nat.ptr(self.feat_lo), nat.ptr(self.post_ord),
                     nat.ptr(self.pnorm2), _sp(stream))
            del X
        del pos
        self._finish(stream, planes_ready=True)
        return self

    @classmethod
    def from_arrays(cls, cb: DeviceCodebook, cell_off: torch.Tensor, post_ord: torch.Tensor,
                    feat: torch.Tensor, n_local: int, n_views: int, ord_base: int = 0,
                    stream=None) -> "DeviceFif":
        """Rebuild from stored lists (load_fif, matching.py:182-211)."""
        self = cls()
        self.cb, self.ord_base, self.n_local, self.V, self.d = cb, int(ord_base), n_local, n_views, cb.d
        self.cell_off = cell_off.to(torch.int64).contiguous()
        self.post_ord = post_ord.to(torch.int32).contiguous()
        self.feat = feat.contiguous()
        self.pnorm2 = (self.feat.double() ** 2).sum(dim=1).float() if self.P else torch.zeros(0, dtype=torch.float32, device=feat.device)
        self._finish(stream)
        return self

    def _finish(self, stream=None, planes_ready: bool = False):
        """Tensor-core operand planes, segments, scan tiles and the shape ->
        postings map."""
        K, P, dev, n_local = self.cb.K, self.P, self.post_ord.device, self.n_local
        if planes_ready:
            pass
        elif P and self.d % 8 == 0:
            if self.feat.dtype == torch.float16:
                self.feat_hi, self.feat_lo = self.feat, None  # exact: no correction plane
            else:
                self.feat_hi = torch.empty((P, self.d), dtype=torch.float16, device=dev)
                self.feat_lo = torch.empty((P, self.d), dtype=torch.float16, device=dev)
                nat.call("gift_split_planes", nat.ptr(self.feat), P * self.d,
                         nat.ptr(self.feat_hi), nat.ptr(self.feat_lo), _sp(stream))
        else:
            self.feat_hi = self.feat_lo = None
        ws = nat.workspace("build", stream).get(nat.lib().gift_fif_build_ws_bytes(P, K))
        self.seg_off = torch.empty(K + 1, dtype=torch.int64, device=dev)
        nat.call("gift_fif_segments", nat.ptr(self.cell_off), nat.ptr(self.post_ord), K, P,
                 nat.ptr(self.seg_off), None, None, nat.ptr(ws), ws.numel(), _sp(stream))
        S = int(self.seg_off[K].item())
        self.S = S
        self.seg_ord = torch.empty(max(S, 1), dtype=torch.int32, device=dev)
        self.seg_pstart = torch.empty(S + 1, dtype=torch.int32, device=dev)
        nat.call("gift_fif_segments", nat.ptr(self.cell_off), nat.ptr(self.post_ord), K, P,
                 nat.ptr(self.seg_off), nat.ptr(self.seg_ord), nat.ptr(self.seg_pstart),
                 nat.ptr(ws), ws.numel(), _sp(stream))
        tile_n = nat.lib().gift_fif_tile_n()
        self.tile_off = torch.empty(K + 1, dtype=torch.int64, device=dev)
        nat.call("gift_fif_tiles", nat.ptr(self.cell_off), nat.ptr(self.seg_off),
                 nat.ptr(self.seg_pstart), K, tile_n, nat.ptr(self.tile_off), None, None, None,
                 None, nat.ptr(ws), ws.numel(), _sp(stream))
        T = int(self.tile_off[K].item())
        self.T = T
        tt = torch.empty((4, max(T, 1)), dtype=torch.int32, device=dev)
        self.tile_pstart, self.tile_pend, self.tile_seg0, self.tile_seg1 = tt[0], tt[1], tt[2], tt[3]
        nat.call("gift_fif_tiles", nat.ptr(self.cell_off), nat.ptr(self.seg_off),
                 nat.ptr(self.seg_pstart), K, tile_n, nat.ptr(self.tile_off),
                 nat.ptr(self.tile_pstart), nat.ptr(self.tile_pend), nat.ptr(self.tile_seg0),
                 nat.ptr(self.tile_seg1), nat.ptr(ws), ws.numel(), _sp(stream))
        # shape -> postings (cell-major order within each shape), index.py:302-314
        k2 = (self.post_ord - self.ord_base).contiguous()
        v2 = torch.arange(P, dtype=torch.int32, device=dev)
        radix_sort_pairs(k2, v2, _bits(n_local), stream)
        self.shape_off = offsets_from_sorted(k2, n_local, stream)  # [n_local+1]
        self.shape_post = v2.to(torch.int64)
        seg_sizes = self.seg_off[1:] - self.seg_off[:-1]
        self.seg_len_max = int((self.seg_pstart[1:S + 1] - self.seg_pstart[:S]).max().item()) if S else 0
        self.smax = int(seg_sizes.max().item()) if K else 0
        # shape -> segments (ascending cell) for the gather reduce: stable sort
        # of the segment indices by owner
        seg_cell = torch.repeat_interleave(
            torch.arange(K, dtype=torch.int32, device=dev), seg_sizes, output_size=S)
        k3 = (self.seg_ord[:S] - self.ord_base).contiguous()
        v3 = torch.arange(S, dtype=torch.int32, device=dev)
        radix_sort_pairs(k3, v3, _bits(n_local), stream)
        self.shape_seg_off = offsets_from_sorted(k3, n_local, stream)  # [n_local+1]
        if S:
            self.shape_seg = v3
            self.shape_seg_cell = seg_cell[v3.long()].contiguous()
            # segments whose shape has no other segment (config 4: every
            # shape's views share one cell): the owner reduce skips the
            # shape's segment lookups (three scattered loads per pair)
            nseg = self.shape_seg_off[1:] - self.shape_seg_off[:-1]
            self.seg_single = (nseg[(self.seg_ord[:S] - self.ord_base).long()] == 1).to(
                torch.uint8).contiguous()
        else:
            self.shape_seg = torch.zeros(1, dtype=torch.int32, device=dev)
            self.shape_seg_cell = torch.zeros(1, dtype=torch.int32, device=dev)
            self.seg_single = torch.zeros(1, dtype=torch.uint8, device=dev)
        self.bind()

    # -- host views (reference container attributes) ---------------------
    def host_lists(self):
        if self.feat is None:
            raise Unsupported("this index keeps only the tensor-core planes on the device "
                              "(streamed build without keep_features): no stored features")
        off = self.cell_off.cpu().numpy()
        ords = self.post_ord.cpu().numpy()
        feats = self.feat.float().cpu().numpy()
        return ([ords[off[c]:off[c + 1]] for c in range(self.cb.K)],
                [feats[off[c]:off[c + 1]] for c in range(self.cb.K)])

    def shape_views(self, local: torch.Tensor):
        """Stored views of shapes (local indices) recovered cell-major, f32,
        zero-padded to the max count; returns (Q [B, Vmax, d], vq [B])."""
        local = local.to(torch.int64)
        starts = self.shape_off[local]
        counts = self.shape_off[local + 1] - starts
        B = local.numel()
        vmax = int(counts.max().item()) if B else 0
        if vmax == 0:
            raise EmptySet("shape has no stored views")
        ar = torch.arange(vmax, device=local.device)
        valid = ar[None, :] < counts[:, None]
        pidx = self.shape_post[(starts[:, None] + ar[None, :]).clamp(max=self.P - 1)]
        rows = torch.where(valid, pidx, torch.full_like(pidx, -1)).reshape(-1)
        Q = torch.zeros((B * vmax, self.d), dtype=torch.float32, device=local.device)
        sel = torch.nonzero(rows >= 0).view(-1)
        if sel.numel():
            tmp = torch.empty((sel.numel(), self.d), dtype=torch.float32, device=local.device)
            src_rows = rows[sel].contiguous()
            if self.feat is not None:
                nat.call("gift_gather_rows_f32", nat.ptr(self.feat), _DTYPE_CODE[self.feat.dtype],
                         self.d, nat.ptr(src_rows), sel.numel(), nat.ptr(tmp), _sp())
            else:
                nat.call("gift_gather_rows_planes", nat.ptr(self.feat_hi), nat.ptr(self.feat_lo),
                         self.d, nat.ptr(src_rows), sel.numel(), nat.ptr(tmp), _sp())
            Q[sel] = tmp
        return Q.view(B, vmax, self.d), counts.to(torch.int32)


class ScoreRunner:
    """K3 launcher with a pre-sized (or grow-on-overflow) compact workspace.

    The compact (probe x segment) buffer is sized for its worst case
    B V ma max_cell_segments whenever that fits the budget (a quarter of the
    HBM free at first use, at most 16 GiB per stream): the batch then never
    needs the host to read the plan's overflow word, so nothing in the query
    path synchronises (config 4's Zipf head cells: ~8 GiB).  Larger bounds
    fall back to a capacity that grows on overflow, checked per batch."""

    MAX_BOUND_BYTES = 16 << 30

    def __init__(self):
        self.capacity = 1 << 22
        self._ws = {}  # stream handle -> Workspace (batches in flight on two streams)
        self._budget = None  # compact floats we are willing to pre-size for

    def score(self, fif: DeviceFif, Q: torch.Tensor, ma: int, mode: int = nat.SIM_COSINE,
              sigma: float = 0.5, vq: torch.Tensor | None = None, out: torch.Tensor | None = None,
              stream=None, scan_events=None, cand_k: int = 0, dense: bool = True,
              reserve_sms: int = 0):
        """Q: [B, V, d] f32 device -> f64 [B, n_local] (matching.py:136-161).
        With cand_k > 0 also returns the reduce's per-range best cand_k
        (scores [B, m], ordinals [B, m]) for `topk_candidates`; with
        dense=False (and cand_k > 0) the dense scores are not written and the
        first returned value is None.  reserve_sms: SMs the scan leaves to the
        kernels of other batches in flight (GIFT_FIF_RESERVE_SMS)."""
        if Q.dim() != 3:
            raise ValueError("queries must be [B, V, d]")
        B, V, d = Q.shape
        if V == 0:
            raise EmptySet("view set is empty")
        if d != fif.d:
            raise DimensionMismatch(f"query dim {d} != index dim {fif.d}")
        if not 1 <= ma <= fif.cb.K:
            raise ValueError(f"ma must be in [1, {fif.cb.K}]")
        Q = Q.contiguous()
        if Q.dtype != torch.float32:
            Q = Q.float()
        if not dense and cand_k <= 0:
            raise ValueError("dense=False needs cand_k > 0")
        if out is None and dense:
            out = torch.empty((B, fif.n_local), dtype=torch.float64, device=Q.device)
        view = fif.view
        if reserve_sms:
            view = type(view).from_buffer_copy(view)
            view.flags = (view.flags & ~0xFF00) | nat.fif_reserve_sms(reserve_sms)
        lib = nat.lib()
        # upper bound of the compact (probe x segment) buffer: if it fits the
        # budget, size for it and skip the host round trip on the overflow flag
        bound = B * V * ma * max(fif.smax, 1)
        if self._budget is None:
            free, _ = torch.cuda.mem_get_info(Q.device)
            self._budget = min(self.MAX_BOUND_BYTES, free // 4) // 4
        checked = bound > self._budget
        if not checked:
            self.capacity = max(self.capacity, bound)
        cs = ci = None
        if cand_k > 0:
            nr = lib.gift_fif_score_ranges2(ctypes.byref(view), V, ma)
            cs = torch.empty((B, nr * cand_k), dtype=torch.float64, device=Q.device)
            ci = torch.empty((B, nr * cand_k), dtype=torch.int32, device=Q.device)
        for _attempt in range(8):
            wsb = lib.gift_fif_score_ws_bytes(ctypes.byref(view), B, V, ma, self.capacity)
            ws = self._ws.setdefault(_sp(stream), nat.Workspace()).get(wsb)
            ev0, ev1 = scan_events if scan_events is not None else (None, None)
            nat.check(lib.gift_fif_score_ex2(ctypes.byref(view), nat.ptr(Q), B, V, nat.ptr(vq), ma,
                                             mode, float(sigma), nat.ptr(out), nat.ptr(ws),
                                             ws.numel(), _sp(stream),
                                             None if ev0 is None else ev0.cuda_event,
                                             None if ev1 is None else ev1.cuda_event,
                                             int(cand_k), nat.ptr(cs), nat.ptr(ci)),
                      "gift_fif_score")
            if not checked:
                return (out, cs, ci) if cand_k > 0 else out
            meta = ws[:64].view(torch.int64)
            status = meta[:3].cpu()
            if int(status[2]) == 0:
                return (out, cs, ci) if cand_k > 0 else out
            self.capacity = int(int(status[1]) * 1.25) + 1024
        raise RuntimeError("F-IF compact buffer kept overflowing")


def topk_candidates(cs: torch.Tensor, ci: torch.Tensor, k: int, positive_only: bool = True,
                    stream=None):
    """K4 merge: best k of per-row candidate lists by (score desc, ordinal asc)."""
    B, m = cs.shape
    idx = torch.empty((B, k), dtype=torch.int32, device=cs.device)
    val = torch.empty((B, k), dtype=torch.float64, device=cs.device)
    nat.call("gift_topk_cand", nat.ptr(cs), nat.ptr(ci), B, m, k, int(positive_only), nat.ptr(idx),
             nat.ptr(val), _sp(stream))
    return idx, val


def topk_rows(scores: torch.Tensor, k: int, *, idrank: torch.Tensor | None = None,
              self_local: torch.Tensor | None = None, ord_base: int = 0,
              positive_only: bool = False, stream=None):
    """K4: best-first (idx global i32, val f64) of each row of [B, n]."""
    B, n = scores.shape
    idx = torch.empty((B, k), dtype=torch.int32, device=scores.device)
    val = torch.empty((B, k), dtype=torch.float64, device=scores.device)
    ws = nat.workspace("topk", stream).get(nat.lib().gift_topk_ws_bytes(B, n, k))
    nat.call("gift_topk_rows_ex", nat.ptr(scores.contiguous()), B, n, k, nat.ptr(idrank),
             nat.ptr(self_local), ord_base, int(positive_only), nat.ptr(idx), nat.ptr(val),
             nat.ptr(ws), ws.numel(), _sp(stream))
    return idx, val


# ------------------------------------------------------------------ activations
@dataclass
class ActRows:
    idx: torch.Tensor   # [n, cap] i32
    val: torch.Tensor   # [n, cap] f64
    cnt: torch.Tensor   # [n] i32
    norm: torch.Tensor  # [n] f64

    @property
    def cap(self) -> int:
        return self.idx.shape[1]

    @property
    def n(self) -> int:
        return self.idx.shape[0]

    @classmethod
    def empty(cls, n: int, cap: int, device) -> "ActRows":
        """Uninitialised rows: every libgift producer (act_from_topk, act_mean,
        act_aggregate) writes all cap slots of a row plus cnt and norm."""
        return cls(torch.empty((n, cap), dtype=torch.int32, device=device),
                   torch.empty((n, cap), dtype=torch.float64, device=device),
                   torch.empty(n, dtype=torch.int32, device=device),
                   torch.empty(n, dtype=torch.float64, device=device))

    def rows(self, a: int, b: int) -> "ActRows":
        return ActRows(self.idx[a:b], self.val[a:b], self.cnt[a:b], self.norm[a:b])

    @classmethod
    def from_host(cls, acts, cap: int | None = None, device=None) -> "ActRows":
        """Pack host SparseActivation-likes (indices/values/norm)."""
        device = device or nat.device()
        n = len(acts)
        sizes = [len(a.indices) for a in acts]
        cap = max(cap or 0, max(sizes) if sizes else 0, 1)
        idx = np.full((n, cap), -1, dtype=np.int32)
        val = np.zeros((n, cap), dtype=np.float64)
        for r, a in enumerate(acts):
            idx[r, :sizes[r]] = a.indices
            val[r, :sizes[r]] = a.values
        return cls(torch.from_numpy(idx).to(device), torch.from_numpy(val).to(device),
                   torch.tensor(sizes, dtype=torch.int32).to(device),
                   torch.tensor([float(a.norm) for a in acts], dtype=torch.float64).to(device))

    def to_host(self):
        idx = self.idx.cpu().numpy()
        val = self.val.cpu().numpy()
        cnt = self.cnt.cpu().numpy()
        norm = self.norm.cpu().numpy()
        return [(idx[r, :cnt[r]].astype(np.int64), val[r, :cnt[r]].copy(), float(norm[r]))
                for r in range(len(cnt))]


def act_from_topk(tidx: torch.Tensor, tval: torch.Tensor, k1: int, out: ActRows | None = None,
                  stream=None) -> ActRows:
    B, kk = tidx.shape
    if out is None:
        out = ActRows.empty(B, max(min(k1, kk), 1), tidx.device)
    nat.call("gift_act_from_topk", nat.ptr(tidx), nat.ptr(tval), B, kk, k1, out.cap,
             nat.ptr(out.idx), nat.ptr(out.val), nat.ptr(out.cnt), nat.ptr(out.norm), _sp(stream))
    return out


def act_mean(raw: ActRows, nbr: torch.Tensor, stream=None) -> ActRows:
    """mean_activation (rerank.py:90-100) of raw rows over each nbr row."""
    B, k2 = nbr.shape
    out = ActRows.empty(B, max(raw.cap * max(k2, 1), 1), nbr.device)
    nat.call("gift_act_mean", nat.ptr(raw.idx), nat.ptr(raw.val), nat.ptr(raw.cnt), raw.cap,
             nat.ptr(nbr.contiguous()), B, k2, out.cap, nat.ptr(out.idx), nat.ptr(out.val),
             nat.ptr(out.cnt), nat.ptr(out.norm), _sp(stream))
    return out


def act_aggregate(a: ActRows, b: ActRows, alpha: float, stream=None) -> ActRows:
    out = ActRows.empty(a.n, a.cap + b.cap, a.idx.device)
    nat.call("gift_act_aggregate", nat.ptr(a.idx), nat.ptr(a.val), nat.ptr(a.cnt), a.cap,
             nat.ptr(b.idx), nat.ptr(b.val), nat.ptr(b.cnt), b.cap, a.n, float(alpha), out.cap,
             nat.ptr(out.idx), nat.ptr(out.val), nat.ptr(out.cnt), nat.ptr(out.norm), _sp(stream))
    return out


# ------------------------------------------------------------------ S-IF
@dataclass
class DeviceSif:
    e_off: torch.Tensor   # [N_global + 1] i64
    e_ord: torch.Tensor   # [nnz] i32 local owner
    e_val: torch.Tensor   # [nnz] f64
    norms: torch.Tensor   # [n_local] f64
    n_global: int
    ord_base: int = 0

    @property
    def n_local(self) -> int:
        return self.norms.numel()

    @classmethod
    def build(cls, final: ActRows, n_global: int, ord_base: int = 0, stream=None) -> "DeviceSif":
        """rerank.py:187-208: transpose of the (local) final activations."""
        dev = final.idx.device
        n = final.n
        row_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        ws = nat.workspace("sif", stream).get((1 << 20) + 16 * n)
        nat.call("gift_act_compact", nat.ptr(final.idx), nat.ptr(final.val), nat.ptr(final.cnt),
                 final.cap, n, nat.ptr(row_off), None, None, None, None, nat.ptr(ws), ws.numel(),
                 _sp(stream))
        nnz = int(row_off[n].item())
        key = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        pos = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        owner = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        nat.call("gift_act_compact", nat.ptr(final.idx), nat.ptr(final.val), nat.ptr(final.cnt),
                 final.cap, n, nat.ptr(row_off), nat.ptr(key), nat.ptr(pos), nat.ptr(owner),
                 nat.ptr(val), nat.ptr(ws), ws.numel(), _sp(stream))
        key, pos = key[:nnz].contiguous(), pos[:nnz].contiguous()
        radix_sort_pairs(key, pos, _bits(n_global), stream)
        e_off = offsets_from_sorted(key, n_global, stream)
        e_ord = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        e_val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        nat.call("gift_sif_permute", nat.ptr(pos), nat.ptr(owner), nat.ptr(val), nnz,
                 nat.ptr(e_ord), nat.ptr(e_val), _sp(stream))
        return cls(e_off, e_ord[:nnz], e_val[:nnz], final.norm.clone(), n_global, ord_base)

    @property
    def max_list(self) -> int:
        """Longest S-IF entry (bounds the shapes one query entry touches)."""
        ml = getattr(self, "_max_list", None)
        if ml is None:
            ml = int((self.e_off[1:] - self.e_off[:-1]).max().item()) if self.n_global else 0
            self._max_list = ml
        return ml

    def _acc_rows(self, B: int, stream=None) -> torch.Tensor:
        """Zeroed f64 accumulator rows for the sparse query (kept zero by the
        kernel): up to 2 per SM, within ~2.5 GB; one set per stream."""
        sms = torch.cuda.get_device_properties(self.norms.device).multi_processor_count
        # row stride: n_local rounded to 64 doubles plus 40 (320 B): rows whose
        # stride is a multiple of a large power of two put the same hot shape
        # of every row on the same DRAM channel (measured 2.3x slower on C5)
        stride = (max(self.n_local, 1) + 63) // 64 * 64 + 40
        want = max(1, min(B, 2 * sms, (2_500_000_000 // 8) // stride))
        pool = self.__dict__.setdefault("_acc", {})
        key = _sp(stream)
        acc = pool.get(key)
        if torch.cuda.is_current_stream_capturing():
            self.__dict__["_acc_captured"] = True
        if acc is None or acc.shape[0] < want:
            if acc is not None and self.__dict__.get("_acc_captured"):
                # a captured CUDA graph still addresses the old rows
                self.__dict__.setdefault("_acc_retired", []).append(acc)
            acc = torch.zeros((want, stride), dtype=torch.float64, device=self.norms.device)
            if stream is not None:
                torch.cuda.current_stream().synchronize()  # zeroed before `stream` uses it
            pool[key] = acc
        return acc

    def query_topk(self, q: ActRows, k: int, order: torch.Tensor, idrank: torch.Tensor | None,
                   self_local: torch.Tensor | None = None, stream=None, flags: int | None = None):
        """Sparse query_sif + final top-k (index.py:290-294): identical to
        topk_rows(self.query(q), k, idrank=..., self_local=...) without the
        dense [B, n] rows.  flags: nat.SIF_ROWS / SIF_SORT / SIF_BUCKET force one
        of the three implementations (default: `self.query_flags`, 0 = by
        batch size)."""
        flags = int(getattr(self, "query_flags", 0) if flags is None else flags)
        B = q.n
        dev = q.idx.device
        idx = torch.empty((B, k), dtype=torch.int32, device=dev)
        val = torch.empty((B, k), dtype=torch.float64, device=dev)
        if B == 0:
            return idx, val
        bound = q.cap * self.max_list
        lib = nat.lib()
        ws = nat.workspace("sif_topk", stream).get(
            lib.gift_sif_query_topk_ws_bytes(B, q.cap, self.n_local, k, bound, flags))
        acc = self._acc_rows(B, stream)
        nat.call("gift_sif_query_topk", nat.ptr(self.e_off), nat.ptr(self.e_ord),
                 nat.ptr(self.e_val), nat.ptr(self.norms), self.n_global, self.n_local,
                 nat.ptr(q.idx), nat.ptr(q.val), nat.ptr(q.cnt), nat.ptr(q.norm), B, q.cap,
                 nat.ptr(acc), acc.shape[0], acc.shape[1], nat.ptr(order), nat.ptr(idrank),
                 nat.ptr(self_local), self.ord_base, k, bound, nat.ptr(idx), nat.ptr(val),
                 nat.ptr(ws), ws.numel(), flags, _sp(stream))
        return idx, val

    def query(self, q: ActRows, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """rerank.py:211-230 for a batch -> dense f64 [B, n_local]."""
        B = q.n
        if out is None:
            out = torch.empty((B, self.n_local), dtype=torch.float64, device=q.idx.device)
        nat.call("gift_sif_query", nat.ptr(self.e_off), nat.ptr(self.e_ord), nat.ptr(self.e_val),
                 nat.ptr(self.norms), self.n_global, self.n_local, nat.ptr(q.idx), nat.ptr(q.val),
                 nat.ptr(q.cnt), nat.ptr(q.norm), B, q.cap, nat.ptr(out), _sp(stream))
        return out

    def host_lists(self):
        off = self.e_off.cpu().numpy()
        o = self.e_ord.cpu().numpy() + self.ord_base
        v = self.e_val.cpu().numpy()
        return ([o[off[i]:off[i + 1]].astype(np.int32) for i in range(self.n_global)],
                [v[off[i]:off[i + 1]].copy() for i in range(self.n_global)])
