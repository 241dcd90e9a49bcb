"""Database sharded by shape across ranks (configs 3-5).

Rank g owns the contiguous ordinal range [g N / G, (g+1) N / G) and holds
that range's postings for every cell (so every cell, including Zipf head
cells, is split evenly) plus the S-IF postings of its own shapes.  Raw
activations (N x k1) are replicated.  Per query batch there are exactly two
exchanges, each ONE `all_gather_into_tensor` of the per-shard best-first
candidates packed as int64 pairs [B, k, 2] = (score bits, ordinal << 32 |
tiebreak), merged on the device by `gift_topk_cand_tb`:

  1. after the F-IF scan: per-shard top-k2 (score, ordinal), key (score desc,
     ordinal asc), positives only (rerank.py:78-87) -- exact, the key is a
     total order and every shard contributes its own best k2;
  2. after the S-IF: per-shard top-k (score, ordinal) by (score desc, own
     entry first, id rank) (index.py:290-294), the zero-score fill coming from
     the shards' own candidates (each shard proposes its best k by the key).

Collectives run on the process group given (NCCL over NVLink on the B200
box; gloo stages through the host in the CPU tests).  All scoring and the
merges stay in libgift kernels.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _native as nat
from . import engine as eg
from .index import CAND_K_MAX

_MISSING_TB = 0xFFFFFFFF


def shard_bounds(n: int, world: int, rank: int):
    """Contiguous, balanced ordinal range of `rank`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def pack_candidates(vals: torch.Tensor, idx: torch.Tensor, tb: torch.Tensor) -> torch.Tensor:
    """[B, k] (f64 score, i32/i64 ordinal, tiebreak < 2^32) -> [B, k, 2] int64:
    (score bits, ordinal << 32 | tiebreak); missing candidates (ordinal < 0)
    keep ordinal -1 and the worst tiebreak."""
    v = vals.to(torch.float64).contiguous().view(torch.int64)
    o = idx.to(torch.int64)
    t = torch.where(o < 0, torch.full_like(o, _MISSING_TB), tb.to(torch.int64) & _MISSING_TB)
    return torch.stack([v, (o << 32) | t], dim=-1)


def unpack_candidates(packed: torch.Tensor):
    """[..., 2] int64 -> (f64 scores, i32 ordinals, i32 tiebreak bits)."""
    v = packed[..., 0].contiguous().view(torch.float64)
    o = (packed[..., 1] >> 32).to(torch.int32)
    t = (packed[..., 1] & _MISSING_TB).to(torch.int32)  # uint32 bits in int32 storage
    return v, o, t


def _all_gather(t: torch.Tensor, group=None) -> torch.Tensor:
    G = dist.get_world_size(group)
    host = t.is_cuda and dist.get_backend(group) == "gloo"  # gloo: stage through host
    src = t.cpu() if host else t.contiguous()
    buf = torch.empty((G * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype,
                      device=src.device)
    dist.all_gather_into_tensor(buf, src, group=group)
    buf = buf.view((G,) + tuple(src.shape))
    return buf.to(t.device) if host else buf


def device_merge(vals, idx, tb, k: int, positive_only: bool, stream=None):
    """Best k per row of [B, m] candidates by (score desc, tiebreak asc)
    (libgift K4 merge)."""
    B, m = vals.shape
    out_i = torch.empty((B, k), dtype=torch.int32, device=vals.device)
    out_v = torch.empty((B, k), dtype=torch.float64, device=vals.device)
    nat.call("gift_topk_cand_tb", nat.ptr(vals.contiguous()), nat.ptr(idx.contiguous()),
             nat.ptr(tb.contiguous()), B, m, k, int(positive_only), nat.ptr(out_i),
             nat.ptr(out_v), nat.stream_ptr(stream))
    return out_i, out_v


def exchange_topk(vals, idx, tb, k: int, positive_only: bool = False, group=None,
                  merge=None):
    """One all_gather_into_tensor of the packed per-shard candidates ([B, k']
    each rank) and the merge into the global best k: returns (idx [B, k] i32,
    -1 padded, vals [B, k] f64).  `merge` defaults to the device kernel (the
    CPU tests pass a host reference merge)."""
    if dist.get_world_size(group) == 1:  # nothing to exchange: merge in place
        return (merge or device_merge)(vals.to(torch.float64).contiguous(),
                                       idx.to(torch.int32).contiguous(),
                                       (tb.to(torch.int64) & _MISSING_TB).to(torch.int32),
                                       k, positive_only)
    packed = _all_gather(pack_candidates(vals, idx, tb), group)  # [G, B, k', 2]
    G, B, kk, _ = packed.shape
    v, o, t = unpack_candidates(packed.permute(1, 0, 2, 3).reshape(B, G * kk, 2))
    return (merge or device_merge)(v, o, t, k, positive_only)


def ordinal_tiebreak(idx: torch.Tensor) -> torch.Tensor:
    """rerank.py:74 / :86 tiebreak: the shape ordinal."""
    return idx.to(torch.int64)


def ranking_tiebreak(idx: torch.Tensor, idrank: torch.Tensor, self_global: torch.Tensor):
    """index.py:290-294 tiebreak: own entry first (0), then 1 + id rank."""
    safe = idx.clamp(min=0).to(torch.int64)
    tb = 1 + idrank.to(torch.int64)[safe]
    return torch.where(idx.to(torch.int64) == self_global.to(torch.int64)[:, None],
                       torch.zeros_like(tb), tb)


def build_sharded(X_local: torch.Tensor, cb: eg.DeviceCodebook, cfg, n_global: int, group=None,
                  batch: int = 256, query_views=None):
    """index.py:185-227 across shards: local F-IF, distributed self-join
    (every shape's views are a query batch on every rank; per-shard top-k
    candidates exchanged and merged), replicated raw activations, local
    co-augment and local S-IF (global coordinates, local owners).

    query_views(s0, s1) -> device views [s1 - s0, V, d] of global shapes
    s0..s1: each rank regenerates (or holds) the self-join's query blocks
    itself; without it the owning rank broadcasts them (f32)."""
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
    nbr = torch.empty((n_global, max(k2, 1)), dtype=torch.int32, device=dev)
    runner = eg.ScoreRunner()
    mode = sim_mode(cfg.similarity)
    V, d = X_local.shape[1], X_local.shape[2]
    for b0 in range(0, n_global, batch):
        b1 = min(n_global, b0 + batch)
        if query_views is not None:
            Q = query_views(b0, b1).float().contiguous()
        else:  # the owners broadcast their rows of this block
            Q = torch.empty((b1 - b0, V, d), dtype=torch.float32, device=dev)
            for r in range(G):
                rlo, rhi = shard_bounds(n_global, G, r)
                s0, s1 = max(b0, rlo), min(b1, rhi)
                if s0 >= s1:
                    continue
                part = (X_local[s0 - lo:s1 - lo].float().contiguous() if r == rank
                        else torch.empty((s1 - s0, V, d), dtype=torch.float32, device=dev))
                _broadcast(part, r, group)
                Q[s0 - b0:s1 - b0] = part
        s = runner.score(fif, Q, cfg.ma, mode, cfg.sigma)
        li, lv = eg.topk_rows(s, kk, positive_only=True, ord_base=lo)  # -1 padded: same shape on every rank
        gi, gv = exchange_topk(lv, li, ordinal_tiebreak(li), kk, True, group)
        eg.act_from_topk(gi, gv, k1, out=raw.rows(b0, b1))
        nbr[b0:b1] = gi[:, : nbr.shape[1]]
    final = eg.act_mean(raw, nbr[lo:hi].contiguous())
    sif = eg.DeviceSif.build(final, n_global, ord_base=lo)
    return fif, raw, sif


def _broadcast(t: torch.Tensor, src: int, group=None) -> torch.Tensor:
    if t.is_cuda and dist.get_backend(group) == "gloo":
        h = t.cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)
    return t


def build_sharded_from_lists(idx: torch.Tensor, val: torch.Tensor, cfg, group=None):
    """Config 5 across shards: the given best-first lists of every shape are
    replicated (each rank generates or loads them), raw activations for all N
    (replicated, as above), the co-augment and the S-IF only for this rank's
    shapes (index.py:211-218)."""
    G = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n, L = idx.shape
    lo, hi = shard_bounds(n, G, rank)
    k1, k2 = min(cfg.k1, L), min(cfg.k2, L)
    raw = eg.act_from_topk(idx, val, k1)
    nbr = torch.where(val[lo:hi, :k2] > 0, idx[lo:hi, :k2],
                      torch.full_like(idx[lo:hi, :k2], -1)).to(torch.int32).contiguous()
    final = eg.act_mean(raw, nbr)
    sif = eg.DeviceSif.build(final, n, ord_base=lo)
    return raw, sif


class ShardedEngine:
    """Query pipeline over one shard with the two cross-shard exchanges.

    `fif` is this rank's DeviceFif (global ordinals; None for a list-only
    index, config 5), `raw` the replicated raw activations (ActRows over all N
    shapes), `sif` this rank's DeviceSif (global coordinates, local owners),
    `idrank` the global id-rank array."""

    def __init__(self, fif, raw: eg.ActRows, sif: eg.DeviceSif, idrank, cfg, n_global: int,
                 group=None):
        self.fif, self.raw, self.sif, self.cfg = fif, raw, sif, cfg
        self.idrank = idrank
        self.n_global = n_global
        self.group = group
        self.runner = eg.ScoreRunner()
        from .matching import sim_mode
        self.mode = sim_mode(cfg.similarity)
        base, n_local = sif.ord_base, sif.n_local
        self.base, self.n_local = base, n_local
        self.idrank_local = idrank[base:base + n_local].contiguous()
        # local shapes in global id-rank order (the sparse S-IF's zero-score fill)
        self.order_local = torch.argsort(self.idrank_local).to(torch.int32).contiguous()

    def _local_self(self, self_global, B, dev):
        if self_global is None:
            self_global = torch.full((B,), -1, dtype=torch.int64, device=dev)
        loc = self_global.to(torch.int64) - self.base
        loc = torch.where((loc >= 0) & (loc < self.n_local), loc,
                          torch.full_like(loc, -1)).to(torch.int32)
        return self_global.to(torch.int64), loc

    def _rank(self, fa: eg.ActRows, k: int, self_global, loc_self):
        if k <= 256:
            li, lv = self.sif.query_topk(fa, k, self.order_local, self.idrank_local, loc_self)
        else:
            li, lv = eg.topk_rows(self.sif.query(fa), k, idrank=self.idrank_local,
                                  self_local=loc_self, ord_base=self.base)
        tb = ranking_tiebreak(li, self.idrank, self_global)
        return exchange_topk(lv, li, tb, k, False, self.group)

    def run(self, Q: torch.Tensor, top_k: int, rerank: bool = True, self_global=None):
        cfg = self.cfg
        B = Q.shape[0]
        self_global, loc_self = self._local_self(self_global, B, Q.device)
        k = min(top_k, self.n_global)
        if rerank:
            k2 = min(cfg.k2, self.n_global)
            if k2 <= CAND_K_MAX:  # local top-k2 straight from the reduce's candidates
                _, cs, ci = self.runner.score(self.fif, Q, cfg.ma, self.mode, cfg.sigma,
                                              cand_k=k2, dense=False)
                li, lv = eg.topk_candidates(cs, ci, k2, positive_only=True)
            else:
                s = self.runner.score(self.fif, Q, cfg.ma, self.mode, cfg.sigma)
                li, lv = eg.topk_rows(s, k2, positive_only=True, ord_base=self.base)
            nbr, _ = exchange_topk(lv, li, ordinal_tiebreak(li), k2, True, self.group)
            return self._rank(eg.act_mean(self.raw, nbr), k, self_global, loc_self)
        s = self.runner.score(self.fif, Q, cfg.ma, self.mode, cfg.sigma)
        li, lv = eg.topk_rows(s, k, idrank=self.idrank_local, self_local=loc_self,
                              ord_base=self.base)
        tb = ranking_tiebreak(li, self.idrank, self_global)
        return exchange_topk(lv, li, tb, k, False, self.group)

    def run_many(self, batches, top_k: int, rerank: bool = True, lanes: int = 2):
        """Query batches in flight on `lanes` streams: batch i runs on stream
        i % lanes (its own scratch), so batch i+1's quantize and scan overlap
        batch i's exchanges and S-IF.  Every rank issues the same batches in
        the same order, so the collectives match.  Returns the per-batch
        (idx, val) on the device."""
        from .index import lane_streams

        main = torch.cuda.current_stream()
        streams = lane_streams(max(1, lanes))
        for st in streams:
            st.wait_stream(main)
        out = []
        for i, Q in enumerate(batches):
            st = streams[i % len(streams)]
            with torch.cuda.stream(st):
                out.append(self.run(Q, top_k, rerank=rerank))
        for st in streams:
            main.wait_stream(st)
        return out

    def rerank_lists(self, q_idx, q_val, top_k: int, self_global=None):
        """Config 5 re-rank from given best-first lists (index.py:249-299):
        the neighbours (first k2 positive entries) are global already, so the
        only exchange is the final ranking's."""
        B = q_idx.shape[0]
        self_global, loc_self = self._local_self(self_global, B, q_idx.device)
        k2 = min(self.cfg.k2, q_idx.shape[1])
        nbr = torch.where(q_val[:, :k2] > 0, q_idx[:, :k2],
                          torch.full_like(q_idx[:, :k2], -1)).to(torch.int32).contiguous()
        return self._rank(eg.act_mean(self.raw, nbr), min(top_k, self.n_global), self_global,
                          loc_self)
