"""Seeded synthetic workloads of BASELINE.json's configs, generated on the
device (the paper's shape benchmarks are not available; these generators
stand in with the configs' shapes, sizes and value distributions).

C1/C2/C3: Gaussian mixture — class means ~ N(mu0, 1) (mu0 = -0.26 gives
about 60% zeros after ReLU at d = 4096), each shape's views =
normalize(relu(mean + 0.3 N(0, 1))), f32.  Queries come from the same
mixture (independent draws).  Codebooks: K distinct database views sampled
without replacement.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Workload:
    name: str
    n_shapes: int
    n_views: int
    dim: int
    n_classes: int
    K: int
    ma: int
    sigma: float
    k1: int
    k2: int
    top_k: int
    n_queries: int
    batch: int
    mu0: float
    storage: str = "float32"


WORKLOADS = {
    "c1": Workload("c1", 1_000, 64, 256, 40, 64, 1, 0.5, 10, 4, 50, 100, 100, 0.0),
    "c2": Workload("c2", 10_000, 64, 4096, 55, 256, 2, 0.5, 10, 4, 100, 1_000, 64, -0.26),
    "c3s": Workload("c3s", 25_000, 64, 4096, 500, 1024, 2, 0.5, 10, 4, 100, 4_096, 256, -0.26),
}


def mixture(w: Workload, seed: int, device, n_queries: int | None = None, block: int = 512):
    """Returns (db [N, V, d], queries [Q, V, d], labels [N]) on `device`."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    means = torch.randn((w.n_classes, w.dim), generator=g, device=device) + w.mu0
    nq = w.n_queries if n_queries is None else n_queries
    total = w.n_shapes + nq
    labels = torch.randint(0, w.n_classes, (total,), generator=g, device=device)
    dt = torch.float16 if w.storage == "float16" else torch.float32
    db = torch.empty((w.n_shapes, w.n_views, w.dim), dtype=dt, device=device)
    qs = torch.empty((nq, w.n_views, w.dim), dtype=torch.float32, device=device)
    for b0 in range(0, total, block):
        b1 = min(total, b0 + block)
        x = means[labels[b0:b1]][:, None, :] + 0.3 * torch.randn(
            (b1 - b0, w.n_views, w.dim), generator=g, device=device)
        x.clamp_(min=0.0)
        n = x.norm(dim=2, keepdim=True)
        x = x / torch.where(n > 0, n, torch.ones_like(n))
        lo, hi = b0, b1
        if hi <= w.n_shapes:
            db[lo:hi] = x.to(dt)
        elif lo >= w.n_shapes:
            qs[lo - w.n_shapes:hi - w.n_shapes] = x.to(dt).float()
        else:
            cut = w.n_shapes - lo
            db[lo:] = x[:cut].to(dt)
            qs[: hi - w.n_shapes] = x[cut:].to(dt).float()
        del x
    return db, qs, labels[: w.n_shapes]


def sample_centroids(db: torch.Tensor, K: int, seed: int) -> torch.Tensor:
    """K distinct non-zero database views (seeded), f32 [K, d]."""
    flat = db.reshape(-1, db.shape[-1])
    g = torch.Generator(device=db.device)
    g.manual_seed(seed)
    perm = torch.randperm(flat.shape[0], generator=g, device=db.device)
    cand = perm[: 4 * K + 16]
    nz = flat[cand].float().abs().sum(dim=1) > 0
    pick = cand[nz][:K]
    pick, _ = torch.sort(pick)
    return flat[pick].float().contiguous()


def shape_ids(n: int, prefix: str = "s"):
    width = max(4, len(str(n)))
    return [f"{prefix}{i:0{width}d}" for i in range(n)]
