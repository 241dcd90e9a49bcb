"""Contextual re-ranking on the GPU: activations, augmentation, aggregation
and the second inverted file.

Mirrors `shapesearch.rerank` (rerank.py:19-323).  `SparseActivation` and
`make_activation` are the host container (as in the reference); every
operation that computes — top-k selection, neighbourhood means, generalized
mean, S-IF transpose and Jaccard scoring — runs in the K4/K5/K6 kernels.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from . import engine as eg
from .errors import FormatError

DEFAULT_K1 = 10
DEFAULT_K2 = 4
DEFAULT_ALPHA = 0.5


def _seq_sum(values) -> float:
    # sequential ascending-coordinate sum (rerank.py:24-31); the kernels use
    # the same order so self-query accumulators equal cached norms bit-exactly
    total = 0.0
    for v in values:
        total += float(v)
    return total


@dataclass(frozen=True)
class SparseActivation:
    """Sparse membership vector over database shape ordinals (rerank.py:34-48)."""

    owner: str
    indices: np.ndarray  # (s,) int64, strictly ascending
    values: np.ndarray   # (s,) float64, positive
    norm: float

    @property
    def support(self) -> int:
        return len(self.indices)

    def items(self):
        return zip(self.indices.tolist(), self.values.tolist())


def make_activation(owner: str, indices, values) -> SparseActivation:
    """rerank.py:51-61 (container constructor)."""
    indices = np.asarray(indices, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    order = np.argsort(indices, kind="stable")
    indices, values = indices[order], values[order]
    keep = values > 0.0
    indices, values = indices[keep], values[keep]
    return SparseActivation(owner=owner, indices=indices, values=values, norm=_seq_sum(values))


class ActivationList:
    """Device-resident activations (engine.ActRows) that read like the
    reference's list[SparseActivation]."""

    def __init__(self, rows: eg.ActRows, owners):
        self.rows = rows
        self.owners = list(owners)
        self._host = None

    def __len__(self):
        return self.rows.n

    def _materialize(self):
        if self._host is None:
            self._host = [SparseActivation(o, i, v, n)
                          for o, (i, v, n) in zip(self.owners, self.rows.to_host())]
        return self._host

    def __getitem__(self, i):
        return self._materialize()[i]

    def __iter__(self):
        return iter(self._materialize())


def _rows(acts) -> eg.ActRows:
    if isinstance(acts, ActivationList):
        return acts.rows
    return eg.ActRows.from_host(list(acts))


def _owners(acts):
    if isinstance(acts, ActivationList):
        return acts.owners
    return [a.owner for a in acts]


def _scores_tensor(scores):
    s = np.asarray(scores, dtype=np.float64)
    return torch.from_numpy(s[None, :].copy()).to(nat.device())


def build_activation(scores, k1: int, owner: str = "") -> SparseActivation:
    """Top-k1 shapes by (score desc, ordinal asc), zero scores dropped
    (rerank.py:64-75)."""
    if k1 < 1:
        raise ValueError("k1 must be >= 1")
    n = len(scores)
    if n == 0:
        return make_activation(owner, [], [])
    k = min(k1, n)
    tidx, tval = eg.topk_rows(_scores_tensor(scores), k, positive_only=True)
    rows = eg.act_from_topk(tidx, tval, k)
    (i, v, nrm), = rows.to_host()
    return SparseActivation(owner, i, v, nrm)


def top_neighbors(scores, k2: int) -> list:
    """Ordinals of the top-k2 positive-score shapes, best first (rerank.py:78-87)."""
    n = len(scores)
    if n == 0 or k2 < 1:
        return []
    tidx, _ = eg.topk_rows(_scores_tensor(scores), min(k2, n), positive_only=True)
    return [int(i) for i in tidx[0].cpu().tolist() if i >= 0]


def _nbr_tensor(neighbor_lists):
    k2 = max([len(x) for x in neighbor_lists] + [1])
    arr = np.full((len(neighbor_lists), k2), -1, dtype=np.int32)
    for r, lst in enumerate(neighbor_lists):
        arr[r, : len(lst)] = lst
    return torch.from_numpy(arr).to(nat.device())


def _wrap(rows: eg.ActRows, owners):
    return [SparseActivation(o, i, v, n) for o, (i, v, n) in zip(owners, rows.to_host())]


def mean_activation(owner: str, activations, neighbor_list) -> SparseActivation:
    """Mean of the neighbours' activations (rerank.py:90-100)."""
    if not neighbor_list:
        return make_activation(owner, [], [])
    out = eg.act_mean(_rows(activations), _nbr_tensor([list(neighbor_list)]))
    return _wrap(out, [owner])[0]


def neighbor_augment(activations, neighbor_lists) -> list:
    """All-at-once neighbourhood means (rerank.py:103-111)."""
    if len(activations) == 0:
        return []
    out = eg.act_mean(_rows(activations), _nbr_tensor(neighbor_lists))
    return _wrap(out, _owners(activations))


def co_augment(acts1, acts2, neighbors1, neighbors2):
    """Cross-channel augmentation (rerank.py:114-125)."""
    if len(acts1) == 0:
        return [], []
    o1 = eg.act_mean(_rows(acts1), _nbr_tensor(neighbors2))
    o2 = eg.act_mean(_rows(acts2), _nbr_tensor(neighbors1))
    return _wrap(o1, _owners(acts1)), _wrap(o2, _owners(acts2))


def aggregate(f1: SparseActivation, f2: SparseActivation,
              alpha: float = DEFAULT_ALPHA) -> SparseActivation:
    """Generalized mean over the union support (rerank.py:128-147)."""
    if alpha <= 0.0:
        raise ValueError("alpha must be > 0")
    out = eg.act_aggregate(eg.ActRows.from_host([f1]), eg.ActRows.from_host([f2]), alpha)
    return _wrap(out, [f1.owner])[0]


def jaccard_dense(fq: SparseActivation, fp: SparseActivation) -> float:
    """Fuzzy Jaccard of two activations (rerank.py:150-162) — the reference's
    brute-force formula, used as a test helper; not on the scoring path."""
    if fq.support == 0 and fp.support == 0:
        return 0.0
    _, qi, pi = np.intersect1d(fq.indices, fp.indices, return_indices=True)
    sum_min = _seq_sum(np.minimum(fq.values[qi], fp.values[pi]))
    sum_max = fq.norm + fp.norm - sum_min
    return 0.0 if sum_max <= 0.0 else sum_min / sum_max


class SecondInvertedFile:
    """Transpose of the database activations plus L1 norms (rerank.py:165-184),
    resident on the GPU (engine.DeviceSif)."""

    def __init__(self, shape_ids, dev: eg.DeviceSif):
        self.shape_ids = list(shape_ids)
        self.dev = dev
        self._host = None

    @property
    def n_shapes(self) -> int:
        return len(self.shape_ids)

    @property
    def norms(self) -> np.ndarray:
        return self.dev.norms.cpu().numpy()

    def _lists(self):
        if self._host is None:
            self._host = self.dev.host_lists()
        return self._host

    @property
    def entry_ordinals(self):
        return self._lists()[0]

    @property
    def entry_values(self):
        return self._lists()[1]

    @property
    def total_postings(self) -> int:
        return int(self.dev.e_ord.numel())


def build_sif(activations, shape_ids=None) -> SecondInvertedFile:
    """rerank.py:187-208 on the GPU (stable radix-sort transpose)."""
    n = len(activations)
    if shape_ids is None:
        shape_ids = _owners(activations)
    if not isinstance(activations, ActivationList):
        for a in activations:
            if len(a.indices) and (a.indices.min() < 0 or a.indices.max() >= n):
                bad = a.indices[(a.indices < 0) | (a.indices >= n)][0]
                raise ValueError(f"activation coordinate {bad} outside database of {n}")
    rows = _rows(activations)
    return SecondInvertedFile(shape_ids, eg.DeviceSif.build(rows, n))


def query_sif(sif: SecondInvertedFile, fq: SparseActivation) -> np.ndarray:
    """Fuzzy Jaccard of one query activation against every shape
    (rerank.py:211-230)."""
    q = eg.ActRows.from_host([fq])
    return sif.dev.query(q)[0].cpu().numpy()


def query_sif_batch(sif: SecondInvertedFile, q: eg.ActRows) -> torch.Tensor:
    return sif.dev.query(q)


# ---------------------------------------------------------------- persistence
def save_sif(sif: SecondInvertedFile, path) -> None:
    """rerank.py:233-244 byte layout."""
    with open(path, "wb") as fh:
        fh.write(struct.pack("<I", sif.n_shapes))
        for sid in sif.shape_ids:
            raw = sid.encode("utf-8")
            fh.write(struct.pack("<H", len(raw)))
            fh.write(raw)
        fh.write(np.asarray(sif.norms).astype("<f8").tobytes())
        for o, v in zip(sif.entry_ordinals, sif.entry_values):
            fh.write(struct.pack("<I", len(o)))
            fh.write(np.asarray(o).astype("<u4").tobytes())
            fh.write(np.asarray(v).astype("<f8").tobytes())


def _reader(path, what):
    data = open(path, "rb").read()
    state = {"off": 0}

    def take(fmt):
        size = struct.calcsize(fmt)
        if state["off"] + size > len(data):
            raise FormatError(f"truncated {what} file {path}")
        out = struct.unpack_from(fmt, data, state["off"])
        state["off"] += size
        return out

    def raw(nbytes):
        if state["off"] + nbytes > len(data):
            raise FormatError(f"truncated {what} file {path}")
        b = data[state["off"]:state["off"] + nbytes]
        state["off"] += nbytes
        return b

    return take, raw


def load_sif(path) -> SecondInvertedFile:
    """rerank.py:247-282: read, rebuild the device CSR."""
    take, raw = _reader(path, "inverted")
    (n,) = take("<I")
    ids = []
    for _ in range(n):
        (ln,) = take("<H")
        ids.append(raw(ln).decode("utf-8"))
    norms = np.frombuffer(raw(8 * n), dtype="<f8").copy()
    counts, ords, vals = [], [], []
    for _ in range(n):
        (c,) = take("<I")
        ords.append(np.frombuffer(raw(4 * c), dtype="<u4").astype(np.int32))
        vals.append(np.frombuffer(raw(8 * c), dtype="<f8").copy())
        counts.append(c)
    dev = nat.device()
    e_off = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int64, device=dev)
    e_ord = torch.from_numpy(np.concatenate(ords) if ords else np.zeros(0, np.int32)).to(dev)
    e_val = torch.from_numpy(np.concatenate(vals) if vals else np.zeros(0)).to(dev)
    d = eg.DeviceSif(e_off, e_ord, e_val, torch.from_numpy(norms).to(dev), n, 0)
    return SecondInvertedFile(ids, d)


def save_activations(activations, path) -> None:
    """rerank.py:285-295 byte layout."""
    acts = list(activations)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<I", len(acts)))
        for a in acts:
            raw = a.owner.encode("utf-8")
            fh.write(struct.pack("<H", len(raw)))
            fh.write(raw)
            fh.write(struct.pack("<I", a.support))
            fh.write(a.indices.astype("<u4").tobytes())
            fh.write(a.values.astype("<f8").tobytes())


def load_activations(path) -> list:
    """rerank.py:298-323."""
    take, raw = _reader(path, "activation")
    (n,) = take("<I")
    out = []
    for _ in range(n):
        (ln,) = take("<H")
        owner = raw(ln).decode("utf-8")
        (c,) = take("<I")
        idx = np.frombuffer(raw(4 * c), dtype="<u4").astype(np.int64)
        val = np.frombuffer(raw(8 * c), dtype="<f8").copy()
        out.append(make_activation(owner, idx, val))
    return out
