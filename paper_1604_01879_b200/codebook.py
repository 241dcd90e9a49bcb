"""Codebook container, the GPU quantizer and codebook training.

Mirrors `shapesearch.codebook` (codebook.py:22-34 Codebook, :37-108
train_codebook, :111-124 quantize, :127-145 persistence).  The benchmark
configs use given codebooks (`sample_codebook`: seeded DB rows, the
BASELINE.json configs' rule, divergence D3); `train_codebook` runs the
reference's k-means++ + Lloyd on the device.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import engine as eg
from .errors import DimensionMismatch, EmptyInput, FormatError

DEFAULT_K = 256
DEFAULT_MAX_ITERS = 50  # codebook.py:18-19
CONVERGENCE_TOL = 1e-4
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


def train_codebook(features, k: int, seed: int = 0, max_iters: int = DEFAULT_MAX_ITERS,
                   channel: str = "") -> Codebook:
    """Lloyd's k-means with k-means++ seeding (codebook.py:48-108).  The host
    runs the reference's control flow and its numpy RNG stream: the same
    draws in the same order (rng.integers for the first center, one
    rng.random per Generator.choice(n, p=...) -- cdf = cumsum(p) / cdf[-1],
    searchsorted(side='right') -- and rng.integers when every distance is
    0), the same empty-cluster repair (largest cluster donates its farthest
    member) and the same relative-cost convergence test.  The device computes
    the f64 distances (gift_kmeans_assign: |x|^2 in numpy's pairwise order,
    the same formula and clamp, ties to the lower index) and the new centers
    (gift_kmeans_update: members summed in point order, np.add.at's order).
    Only the x.c dot products are summed in another order than the
    reference's BLAS, so a label can differ only for a point equidistant to
    two centers within a few ulps."""
    from . import _native as nat

    dev = nat.device()
    if torch.is_tensor(features):  # device rows stay on the device
        X = features.to(dev, torch.float64)
    else:
        X = torch.from_numpy(np.ascontiguousarray(np.asarray(features, dtype=np.float64))).to(dev)
    if X.dim() != 2 or X.shape[0] == 0:
        raise EmptyInput("no training vectors")
    n, d = X.shape
    if n < k:
        X = X.repeat(-(-k // n), 1)  # duplicate inputs up to >= k points (np.tile)
        n = X.shape[0]
    X = X.contiguous()
    xn2 = torch.empty(n, dtype=torch.float64, device=dev)
    nat.call("gift_rows_sqnorm_f64", nat.ptr(X), n, d, nat.ptr(xn2), nat.stream_ptr())
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    mind2 = torch.empty(n, dtype=torch.float64, device=dev)

    def assign(C, want_labels=True):
        C = C.contiguous()
        cn2 = torch.empty(C.shape[0], dtype=torch.float64, device=dev)
        nat.call("gift_rows_sqnorm_f64", nat.ptr(C), C.shape[0], d, nat.ptr(cn2),
                 nat.stream_ptr())
        nat.call("gift_kmeans_assign", nat.ptr(X), n, d, nat.ptr(C), C.shape[0], nat.ptr(xn2),
                 nat.ptr(cn2), nat.ptr(labels) if want_labels else None, nat.ptr(mind2),
                 nat.stream_ptr())
        return mind2.cpu().numpy()

    # k-means++ (codebook.py:48-61)
    rng = np.random.default_rng(seed)
    centers = torch.empty((k, d), dtype=torch.float64, device=dev)
    centers[0] = X[int(rng.integers(0, n))]
    closest = assign(centers[:1], want_labels=False)
    for i in range(1, k):
        total = closest.sum()
        if total <= 0.0:
            idx = int(rng.integers(0, n))
        else:
            cdf = (closest / total).cumsum()  # Generator.choice(n, p=closest / total)
            cdf /= cdf[-1]
            idx = int(cdf.searchsorted(rng.random(), side="right"))
        centers[i] = X[idx]
        np.minimum(closest, assign(centers[i:i + 1], want_labels=False), out=closest)
    # Lloyd (codebook.py:76-104)
    C = centers
    prev_cost = None
    for _ in range(max_iters):
        d2min = assign(C)
        lab = labels.cpu().numpy().astype(np.int64)
        cost = float(d2min.sum())
        counts = np.bincount(lab, minlength=k)
        for empty in np.flatnonzero(counts == 0):
            donor = int(counts.argmax())
            members = np.flatnonzero(lab == donor)
            dd = np.empty(len(members))
            Cd = C[donor:donor + 1].contiguous()
            cn2 = torch.empty(1, dtype=torch.float64, device=dev)
            nat.call("gift_rows_sqnorm_f64", nat.ptr(Cd), 1, d, nat.ptr(cn2), nat.stream_ptr())
            sub = X[torch.from_numpy(members).to(dev)].contiguous()
            sub_n2 = xn2[torch.from_numpy(members).to(dev)].contiguous()
            out = torch.empty(len(members), dtype=torch.float64, device=dev)
            nat.call("gift_kmeans_assign", nat.ptr(sub), len(members), d, nat.ptr(Cd), 1,
                     nat.ptr(sub_n2), nat.ptr(cn2), None, nat.ptr(out), nat.stream_ptr())
            dd[:] = out.cpu().numpy()
            steal = members[dd.argmax()]
            lab[steal] = empty
            counts[donor] -= 1
            counts[empty] += 1
        order = torch.from_numpy(np.argsort(lab, kind="stable")).to(dev)
        off = torch.from_numpy(np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)).to(dev)
        newC = torch.empty((k, d), dtype=torch.float64, device=dev)
        nat.call("gift_kmeans_update", nat.ptr(X), n, d, nat.ptr(order), nat.ptr(off), k,
                 nat.ptr(newC), nat.stream_ptr())
        C = newC
        if prev_cost is not None:
            denom = max(prev_cost, 1e-300)
            if abs(prev_cost - cost) / denom < CONVERGENCE_TOL:
                break
        prev_cost = cost
    cb = Codebook(centroids=C.cpu().numpy().astype(np.float32), channel=channel, seed=seed)
    if np.isnan(cb.centroids).any():
        raise EmptyInput("k-means produced NaN centroids")
    return cb


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
