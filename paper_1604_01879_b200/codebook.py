"""Codebook container and the GPU quantizer.

Mirrors `shapesearch.codebook` (codebook.py:22-34 Codebook, :111-124
quantize, :127-145 persistence).  Codebook training (k-means, codebook.py:37-108)
is outside the GPU path (divergence D3): codebooks are given,
e.g. `sample_codebook` (seeded DB rows, the BASELINE.json configs' rule).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import engine as eg
from .errors import DimensionMismatch, EmptyInput, FormatError

DEFAULT_K = 256
_DEV_CACHE: dict = {}


@dataclass(frozen=True)
class Codebook:
    centroids: np.ndarray  # (K, d) float32
    channel: str = ""
    seed: int = 0

    @property
    def k(self) -> int:
        return self.centroids.shape[0]

    @property
    def dim(self) -> int:
        return self.centroids.shape[1]

    def device(self) -> eg.DeviceCodebook:
        """Device copy (centroids f32, |c|^2 f64), cached per codebook object."""
        key = id(self)
        hit = _DEV_CACHE.get(key)
        if hit is None or hit[0] is not self:
            hit = (self, eg.DeviceCodebook.from_numpy(self.centroids))
            _DEV_CACHE[key] = hit
        return hit[1]


def sample_codebook(vectors, k: int, seed: int = 0, channel: str = "") -> Codebook:
    """K distinct non-zero rows drawn without replacement (seeded)."""
    flat = np.asarray(vectors, dtype=np.float32).reshape(-1, np.asarray(vectors).shape[-1])
    nz = np.flatnonzero(flat.any(axis=1))
    if len(nz) == 0:
        raise EmptyInput("no training vectors")
    rng = np.random.default_rng(seed)
    pick = rng.choice(nz, size=k, replace=len(nz) < k)
    return Codebook(centroids=flat[np.sort(pick)].copy(), channel=channel, seed=seed)


def quantize(codebook: Codebook, x, ma: int = 1) -> np.ndarray:
    """Indices of the ma nearest centroids, ascending by squared distance,
    ties toward the lower index (codebook.py:111-124), computed by the K1
    kernel bit-identically to the reference's f64 pairwise-summed distances."""
    x = np.asarray(x, dtype=np.float64).ravel()
    if x.shape[0] != codebook.dim:
        raise DimensionMismatch(f"vector dim {x.shape[0]} != codebook dim {codebook.dim}")
    if not 1 <= ma <= codebook.k:
        raise ValueError(f"ma must be in [1, {codebook.k}]")
    cb = codebook.device()
    X = torch.from_numpy(x[None, :].copy()).to(cb.centroids.device)
    return eg.quantize_rows(cb, X, ma).cpu().numpy()[0].astype(np.int64)


def quantize_batch(codebook: Codebook, X, ma: int = 1) -> np.ndarray:
    """Row-wise `quantize` for an (n, d) array or device tensor (new API)."""
    cb = codebook.device()
    if not torch.is_tensor(X):
        arr = np.asarray(X)
        X = torch.from_numpy(np.ascontiguousarray(
            arr if arr.dtype in (np.float32, np.float16) else arr.astype(np.float64)))
    X = X.to(cb.centroids.device)
    if X.dim() != 2 or X.shape[1] != codebook.dim:
        raise DimensionMismatch("expected (n, d) vectors matching the codebook")
    return eg.quantize_rows(cb, X, ma).cpu().numpy().astype(np.int64)


def save_codebook(codebook: Codebook, path) -> None:
    """codebook.py:127-132 layout: <IIqH header, channel, f32 centroids."""
    with open(path, "wb") as fh:
        ch = codebook.channel.encode("utf-8")
        fh.write(struct.pack("<IIqH", codebook.k, codebook.dim, codebook.seed, len(ch)))
        fh.write(ch)
        fh.write(np.asarray(codebook.centroids).astype("<f4").tobytes())


def load_codebook(path) -> Codebook:
    data = open(path, "rb").read()
    head = struct.calcsize("<IIqH")
    if len(data) < head:
        raise FormatError(f"truncated codebook file {path}")
    k, dim, seed, n = struct.unpack_from("<IIqH", data, 0)
    channel = data[head:head + n].decode("utf-8")
    body = np.frombuffer(data, dtype="<f4", count=k * dim, offset=head + n) \
        if len(data) >= head + n + 4 * k * dim else np.zeros(0, dtype=np.float32)
    if body.size != k * dim:
        raise FormatError(f"truncated codebook file {path}")
    return Codebook(centroids=body.reshape(k, dim).copy(), channel=channel, seed=seed)
