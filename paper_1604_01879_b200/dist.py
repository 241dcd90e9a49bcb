"""Database sharded by shape across ranks (configs 3-5).

Rank g owns the contiguous ordinal range [g N / G, (g+1) N / G) and holds
that range's postings for every cell (so every cell, including Zipf head
cells, is split evenly) plus the S-IF postings of its own shapes.  Raw
activations (N x k1) are replicated.  Per query batch there are exactly two
exchanges, both `all_gather_into_tensor` of per-shard top-k candidates:

  1. after the F-IF scan: per-shard top-k2 (score, ordinal) -> merged by
     (score desc, ordinal asc) — exact, the key is a total order and every
     shard contributes its own best k2;
  2. after the S-IF: per-shard top-k (score, ordinal) -> merged by
     (score desc, not_self, id rank) with the zero-score fill coming from the
     shards' own candidates (each shard proposes its best k by the same key).

Collectives run on the process group given (NCCL over NVLink on the B200
box, gloo in the CPU tests); the merges are tiny (B x G x k) torch
reductions.  All scoring stays in the libgift kernels.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import engine as eg
from .index import CAND_K_MAX


def shard_bounds(n: int, world: int, rank: int):
    """Contiguous, balanced ordinal range of `rank`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def merge_candidates(vals: torch.Tensor, idx: torch.Tensor, tb: torch.Tensor, k: int):
    """vals/idx/tb: [G, B, k'] per-shard best-first candidates (idx -1 = none).
    Returns the global best k per row by (score desc, tiebreak asc)."""
    G, B, kk = vals.shape
    v = vals.permute(1, 0, 2).reshape(B, G * kk)
    i = idx.permute(1, 0, 2).reshape(B, G * kk)
    t = tb.permute(1, 0, 2).reshape(B, G * kk).to(torch.int64)
    missing = i < 0
    v = torch.where(missing, torch.full_like(v, float("-inf")), v)
    t = torch.where(missing, torch.full_like(t, 1 << 40), t)
    o1 = torch.sort(t, dim=1, stable=True).indices
    v1 = torch.gather(v, 1, o1)
    o2 = torch.sort(v1, dim=1, descending=True, stable=True).indices
    order = torch.gather(o1, 1, o2)[:, :k]
    out_i = torch.gather(i, 1, order)
    out_v = torch.gather(v, 1, order)
    out_i = torch.where(torch.isinf(out_v), torch.full_like(out_i, -1), out_i)
    out_v = torch.where(torch.isinf(out_v), torch.zeros_like(out_v), out_v)
    return out_i, out_v


def _all_gather(t: torch.Tensor, group=None) -> torch.Tensor:
    G = dist.get_world_size(group)
    host = t.is_cuda and dist.get_backend(group) == "gloo"  # gloo: stage through host
    src = t.cpu() if host else t.contiguous()
    buf = torch.empty((G * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype,
                      device=src.device)
    dist.all_gather_into_tensor(buf, src, group=group)
    buf = buf.view((G,) + tuple(src.shape))
    return buf.to(t.device) if host else buf


def all_gather_topk(vals: torch.Tensor, idx: torch.Tensor, tb: torch.Tensor, k: int, group=None):
    """Exchange per-shard candidates ([B, k'] each) and merge (one
    all_gather_into_tensor per array)."""
    outs = [_all_gather(t, group) for t in (vals, idx, tb)]
    return merge_candidates(outs[0], outs[1], outs[2], k)


def _broadcast(t: torch.Tensor, src: int, group=None) -> torch.Tensor:
    if t.is_cuda and dist.get_backend(group) == "gloo":
        h = t.cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)
    return t


def build_sharded(X_local: torch.Tensor, cb: eg.DeviceCodebook, cfg, n_global: int, group=None,
                  batch: int = 256):
    """index.py:185-227 across shards: local F-IF, distributed self-join
    (every shard's shapes are broadcast as query batches; per-shard top-k
    candidates merged), replicated raw activations, local co-augment and
    local S-IF (global coordinates, local owners)."""
    from .matching import sim_mode

    G = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_bounds(n_global, G, rank)
    assert X_local.shape[0] == hi - lo
    fif = eg.DeviceFif.build(X_local, cb, ord_base=lo)
    k1 = min(cfg.k1, n_global)
    k2 = min(cfg.k2, n_global)
    kk = max(k1, k2)
    dev = X_local.device
    raw = eg.ActRows.empty(n_global, max(k1, 1), dev)
    nbr = torch.full((n_global, max(k2, 1)), -1, dtype=torch.int32, device=dev)
    runner = eg.ScoreRunner()
    mode = sim_mode(cfg.similarity)
    V, d = X_local.shape[1], X_local.shape[2]
    for r in range(G):
        rlo, rhi = shard_bounds(n_global, G, r)
        for b0 in range(rlo, rhi, batch):
            b1 = min(rhi, b0 + batch)
            Q = (X_local[b0 - lo:b1 - lo].float().contiguous() if r == rank
                 else torch.empty((b1 - b0, V, d), dtype=torch.float32, device=dev))
            _broadcast(Q, r, group)
            s = runner.score(fif, Q, cfg.ma, mode, cfg.sigma)
            li, lv = eg.topk_rows(s, kk, positive_only=True, ord_base=lo)  # -1 padded: same shape on every rank
            gi, gv = all_gather_topk(lv, li, ordinal_tiebreak(li), kk, group)
            gi = gi.to(torch.int32).contiguous()
            eg.act_from_topk(gi, gv.contiguous(), k1, out=raw.rows(b0, b1))
            nbr[b0:b1] = gi[:, : nbr.shape[1]]
    final = eg.act_mean(raw, nbr[lo:hi].contiguous())
    sif = eg.DeviceSif.build(final, n_global, ord_base=lo)
    return fif, raw, sif


def ordinal_tiebreak(idx: torch.Tensor) -> torch.Tensor:
    """rerank.py:74 / :86 tiebreak: the shape ordinal."""
    return torch.where(idx < 0, torch.full_like(idx, 2**31 - 1), idx).to(torch.int64)


def ranking_tiebreak(idx: torch.Tensor, idrank: torch.Tensor, self_global: torch.Tensor):
    """index.py:290-294 tiebreak: own entry first, then shape-id order."""
    safe = idx.clamp(min=0).to(torch.int64)
    tb = 1 + idrank.to(torch.int64)[safe]
    tb = torch.where(idx.to(torch.int64) == self_global.to(torch.int64)[:, None],
                     torch.zeros_like(tb), tb)
    return torch.where(idx < 0, torch.full_like(tb, 1 << 40), tb)


class ShardedEngine:
    """Query pipeline over one shard with the two cross-shard exchanges.

    `fif` is this rank's DeviceFif (global ordinals), `raw` the replicated
    raw activations (ActRows over all N shapes), `sif` this rank's DeviceSif
    (global coordinates, local owners), `idrank` the global id-rank array."""

    def __init__(self, fif: eg.DeviceFif, raw: eg.ActRows, sif: eg.DeviceSif, idrank, cfg,
                 n_global: int, group=None):
        self.fif, self.raw, self.sif, self.cfg = fif, raw, sif, cfg
        self.idrank = idrank
        self.n_global = n_global
        self.group = group
        self.runner = eg.ScoreRunner()
        from .matching import sim_mode
        self.mode = sim_mode(cfg.similarity)
        base, n_local = fif.ord_base, fif.n_local
        self.idrank_local = idrank[base:base + n_local].contiguous()
        # local shapes in global id-rank order (the sparse S-IF's zero-score fill)
        self.order_local = torch.argsort(self.idrank_local).to(torch.int32).contiguous()

    def run(self, Q: torch.Tensor, top_k: int, rerank: bool = True, self_global=None):
        cfg = self.cfg
        B = Q.shape[0]
        dev = Q.device
        if self_global is None:
            self_global = torch.full((B,), -1, dtype=torch.int64, device=dev)
        base = self.fif.ord_base
        k = min(top_k, self.n_global)
        loc_self = (self_global - base)
        loc_self = torch.where((loc_self >= 0) & (loc_self < self.fif.n_local), loc_self,
                               torch.full_like(loc_self, -1)).to(torch.int32)
        if rerank:
            k2 = min(cfg.k2, self.n_global)
            if k2 <= CAND_K_MAX:  # local top-k2 straight from the reduce's candidates
                _, cs, ci = self.runner.score(self.fif, Q, cfg.ma, self.mode, cfg.sigma,
                                              cand_k=k2, dense=False)
                li, lv = eg.topk_candidates(cs, ci, k2, positive_only=True)
            else:
                s = self.runner.score(self.fif, Q, cfg.ma, self.mode, cfg.sigma)
                li, lv = eg.topk_rows(s, k2, positive_only=True, ord_base=base)
            nbr, _ = all_gather_topk(lv, li, ordinal_tiebreak(li), k2, self.group)
            fa = eg.act_mean(self.raw, nbr.to(torch.int32).contiguous())
            if k <= 256:
                li, lv = self.sif.query_topk(fa, k, self.order_local, self.idrank_local, loc_self)
            else:
                li, lv = eg.topk_rows(self.sif.query(fa), k, idrank=self.idrank_local,
                                      self_local=loc_self, ord_base=base)
        else:
            s = self.runner.score(self.fif, Q, cfg.ma, self.mode, cfg.sigma)
            li, lv = eg.topk_rows(s, k, idrank=self.idrank_local, self_local=loc_self,
                                  ord_base=base)
        tb = ranking_tiebreak(li, self.idrank, self_global)
        return all_gather_topk(lv, li, tb, k, self.group)
