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
    # config 3: 105 GB of f32 views on one GPU -> streamed build, planes only
    "c3": Workload("c3", 100_000, 64, 4096, 500, 1024, 2, 0.5, 10, 4, 100, 4_096, 256, -0.26),
    "c3s": Workload("c3s", 25_000, 64, 4096, 500, 1024, 2, 0.5, 10, 4, 100, 4_096, 256, -0.26),
    # config 4: 1M shapes x 20 views, d=1024 fp16, Zipf(1.1) cell occupancy over
    # K=4096 (classes biased toward Zipf-chosen centroids), ma=1
    "c4": Workload("c4", 1_000_000, 20, 1024, 16_384, 4096, 1, 0.5, 10, 4, 10, 8_192, 512, -0.26,
                   "float16"),
    # reduced config 4 for the 1-GPU tests
    "c4s": Workload("c4s", 50_000, 20, 1024, 4_096, 4096, 1, 0.5, 10, 4, 10, 1_024, 512, -0.26,
                    "float16"),
}

# config 5: re-rank dominated, given top-50 lists (no F-IF stage)
C5 = dict(n_shapes=1_000_000, list_len=50, communities=2_000, noise=0.10, k2=4, top_k=100,
          n_queries=16_384, batch=512)


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


class BlockMixture:
    """Config-3-scale mixture generated block by block: block b of `block`
    shapes is drawn from its own seeded generator, so any shape range can be
    regenerated on the device on demand (the streamed build reads the
    database three times and never holds it whole).  Same distribution as
    `mixture`: views = normalize(relu(mean[label] + 0.3 N(0, 1)))."""

    def __init__(self, w: Workload, seed: int, device, block: int = 256):
        self.w, self.seed, self.device, self.block = w, seed, device, block
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        self.means = torch.randn((w.n_classes, w.dim), generator=g, device=device) + w.mu0
        self.labels = torch.randint(0, w.n_classes, (w.n_shapes + w.n_queries,), generator=g,
                                    device=device)

    def _block(self, b: int) -> torch.Tensor:
        w = self.w
        total = w.n_shapes + w.n_queries
        b0, b1 = b * self.block, min(total, (b + 1) * self.block)
        g = torch.Generator(device=self.device)
        g.manual_seed(self.seed * 1_000_003 + 7919 * b + 1)
        x = self.means[self.labels[b0:b1]][:, None, :] + 0.3 * torch.randn(
            (b1 - b0, w.n_views, w.dim), generator=g, device=self.device)
        x.clamp_(min=0.0)
        n = x.norm(dim=2, keepdim=True)
        return x / torch.where(n > 0, n, torch.ones_like(n))

    def rows(self, s0: int, s1: int) -> torch.Tensor:
        """Views of global rows s0..s1 (database rows, then query rows), f32."""
        out = torch.empty((s1 - s0, self.w.n_views, self.w.dim), dtype=torch.float32,
                          device=self.device)
        b = s0 // self.block
        while b * self.block < s1:
            x = self._block(b)
            lo = max(s0, b * self.block)
            hi = min(s1, (b + 1) * self.block)
            out[lo - s0:hi - s0] = x[lo - b * self.block:hi - b * self.block]
            del x
            b += 1
        return out

    def provider(self, base: int = 0):
        """provider(s0, s1) over database shapes base + s0 .. base + s1."""
        return lambda s0, s1: self.rows(base + s0, base + s1)

    def queries(self) -> torch.Tensor:
        return self.rows(self.w.n_shapes, self.w.n_shapes + self.w.n_queries)


def sample_centroids_rows(mix: "BlockMixture", K: int, seed: int) -> torch.Tensor:
    """`sample_centroids` without the whole database: the same seeded
    permutation over all n_shapes x V views, the first K non-zero candidates
    in permutation order, returned sorted by view index.  Each block holding
    a candidate is generated once."""
    w = mix.w
    V = w.n_views
    g = torch.Generator(device=mix.device)
    g.manual_seed(seed)
    perm = torch.randperm(w.n_shapes * V, generator=g, device=mix.device)
    cand = perm[: 4 * K + 16].tolist()
    rows = {}
    by_block = {}
    for v in cand:
        by_block.setdefault((v // V) // mix.block, []).append(v)
    for b, vs in by_block.items():
        x = mix._block(b)
        for v in vs:
            rows[v] = x[v // V - b * mix.block, v % V].clone()
        del x
    nz = [v for v in cand if float(rows[v].abs().sum()) > 0][:K]
    return torch.stack([rows[v] for v in sorted(nz)]).float().contiguous()


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


def zipf_mixture(w: Workload, seed: int, device, s_exp: float = 1.1, block: int = 4096):
    """Config 4: K centroids ~ normalize(relu(N(mu0, 1))); each class mean is a
    Zipf(s)-chosen centroid's pre-activation plus 0.25 N(0, 1), so the cell
    occupancy follows Zipf(s) over a seeded rank -> cell permutation; views =
    normalize(relu(class + 0.3 N(0, 1))) stored as fp16.  Returns (db, queries,
    centroids f32)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    pre_c = torch.randn((w.K, w.dim), generator=g, device=device) + w.mu0
    cent = pre_c.clamp(min=0.0)
    cent = cent / cent.norm(dim=1, keepdim=True).clamp(min=1e-30)
    ranks = torch.arange(1, w.K + 1, device=device, dtype=torch.float64)
    p = ranks.pow(-s_exp)
    p = p / p.sum()
    cell_of_rank = torch.randperm(w.K, generator=g, device=device)
    cls_rank = torch.multinomial(p.float(), w.n_classes, replacement=True, generator=g)
    cls_pre = pre_c[cell_of_rank[cls_rank]] + 0.25 * torch.randn(
        (w.n_classes, w.dim), generator=g, device=device)
    total = w.n_shapes + w.n_queries
    labels = torch.randint(0, w.n_classes, (total,), generator=g, device=device)
    db = torch.empty((w.n_shapes, w.n_views, w.dim), dtype=torch.float16, device=device)
    qs = torch.empty((w.n_queries, w.n_views, w.dim), dtype=torch.float32, device=device)
    for b0 in range(0, total, block):
        b1 = min(total, b0 + block)
        x = cls_pre[labels[b0:b1]][:, None, :] + 0.3 * torch.randn(
            (b1 - b0, w.n_views, w.dim), generator=g, device=device)
        x.clamp_(min=0.0)
        n = x.norm(dim=2, keepdim=True)
        x = (x / torch.where(n > 0, n, torch.ones_like(n))).to(torch.float16)
        for lo, hi, dst, off in ((b0, min(b1, w.n_shapes), db, 0),
                                 (max(b0, w.n_shapes), b1, qs, w.n_shapes)):
            if hi > lo:
                dst[lo - off:hi - off] = x[lo - b0:hi - b0].to(dst.dtype)
        del x
    return db, qs, cent.float().contiguous()


def community_lists(seed: int, device, n_shapes=C5["n_shapes"], list_len=C5["list_len"],
                    communities=C5["communities"], noise=C5["noise"]):
    """Config 5: per shape a top-`list_len` neighbour list — (1 - noise) of it
    uniform within the shape's community, the rest uniform over all shapes,
    without duplicates — with scores U(0, 1) sorted descending (assigned to a
    random permutation of the list).  Returns (idx [N, L] i32, scores [N, L]
    f64), best first."""
    if n_shapes < 4 * communities * list_len:
        raise ValueError("communities too small for duplicate-free lists: use about "
                         f"{n_shapes // (4 * list_len)} or fewer for {n_shapes} shapes")
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    comm = torch.randint(0, communities, (n_shapes,), generator=g, device=device)
    order = torch.argsort(comm)
    counts = torch.bincount(comm, minlength=communities)
    starts = torch.cumsum(counts, 0) - counts
    n_in = int(round(list_len * (1.0 - noise)))
    n_out = list_len - n_in
    idx = torch.empty((n_shapes, list_len), dtype=torch.int64, device=device)
    blk = 65536
    for b0 in range(0, n_shapes, blk):
        b1 = min(n_shapes, b0 + blk)
        c = comm[b0:b1]
        sz = counts[c].clamp(min=1)
        draw = torch.floor(torch.rand((b1 - b0, 2 * list_len), generator=g, device=device,
                                      dtype=torch.float64) * sz[:, None]).long()
        cand = order[starts[c][:, None] + draw]
        glob = torch.randint(0, n_shapes, (b1 - b0, 2 * list_len), generator=g, device=device)
        both = torch.cat([cand, glob], dim=1)
        # dedupe per row: sort, flag repeats, keep first n_in in-community and
        # n_out global picks in draw order
        srt, pos = torch.sort(both, dim=1, stable=True)
        dup = torch.zeros_like(srt, dtype=torch.bool)
        dup[:, 1:] = srt[:, 1:] == srt[:, :-1]
        keep = torch.ones_like(both, dtype=torch.bool)
        keep.scatter_(1, pos, ~dup)
        key_in = torch.where(keep[:, :2 * list_len], torch.arange(2 * list_len, device=device),
                             torch.full_like(draw, 1 << 30))
        key_gl = torch.where(keep[:, 2 * list_len:], torch.arange(2 * list_len, device=device),
                             torch.full_like(draw, 1 << 30))
        sel_in = torch.argsort(key_in, dim=1, stable=True)[:, :n_in]
        sel_gl = torch.argsort(key_gl, dim=1, stable=True)[:, :n_out]
        rows = torch.cat([torch.gather(cand, 1, sel_in), torch.gather(glob, 1, sel_gl)], dim=1)
        perm = torch.argsort(torch.rand(rows.shape, generator=g, device=device), dim=1)
        idx[b0:b1] = torch.gather(rows, 1, perm)
    scores = torch.sort(torch.rand((n_shapes, list_len), generator=g, device=device,
                                   dtype=torch.float64), dim=1, descending=True).values
    return idx.to(torch.int32), scores
