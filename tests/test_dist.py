"""Shard-by-shape merge logic (dist.py) on CPU with world_size 2 (gloo):
per-shard top-k candidates exchanged with all_gather_into_tensor and merged
must equal the global lexsort selection of the reference (rerank.py:74,
:86-87; index.py:290-294), including ties, zero-score fill and self-first."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_01879_b200.dist import (exchange_topk, ordinal_tiebreak, pack_candidates,
                                        ranking_tiebreak, shard_bounds, unpack_candidates)


def host_merge(v, o, t, k, positive_only):
    """Reference merge of the exchanged candidates (the device kernel's
    contract, gift_topk_cand_tb): best k by (score desc, uint32 tiebreak
    asc), absent entries (ordinal < 0) skipped, -1 / 0.0 padded."""
    B = v.shape[0]
    out_i = torch.full((B, k), -1, dtype=torch.int32)
    out_v = torch.zeros((B, k), dtype=torch.float64)
    for b in range(B):
        vv, oo = v[b].numpy(), o[b].numpy()
        tt = t[b].numpy().astype(np.int64) & 0xFFFFFFFF
        keep = np.flatnonzero(oo >= 0)
        order = keep[np.lexsort((tt[keep], -vv[keep]))][:k]
        for j, x in enumerate(order):
            if positive_only and not vv[x] > 0:
                continue
            out_i[b, j] = int(oo[x])
            out_v[b, j] = vv[x]
    return out_i, out_v


def all_gather_topk(vals, idx, tb, k, positive_only=False):
    return exchange_topk(vals, idx, tb, k, positive_only, merge=host_merge)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _local_topk(S, lo, hi, k, tb_of):
    """Per-shard best k by (score desc, tiebreak asc) — stand-in for the
    K4 kernel on the shard's columns."""
    B = S.shape[0]
    kk = min(k, hi - lo)
    vals = np.zeros((B, k))  # k per rank, -1 padded (uniform all_gather shapes)
    idx = np.full((B, k), -1, dtype=np.int64)
    for b in range(B):
        cols = np.arange(lo, hi)
        tb = np.array([tb_of(b, j) for j in cols])
        order = np.lexsort((tb, -S[b, lo:hi]))[:kk]
        vals[b, :kk] = S[b, lo + order]
        idx[b, :kk] = lo + order
    return vals, idx


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        B, N = 6, 103
        S = np.round(rng.random((B, N)), 2)
        S[:, ::4] = 0.0
        S[2] = 0.0  # an all-zero row: pure zero-fill
        idrank = rng.permutation(N)
        self_global = np.array([5, -1, 50, 102, -1, 0])
        lo, hi = shard_bounds(N, world, rank)
        ok = []
        # (1) neighbour / activation selection: tiebreak = ordinal
        for k in (1, 4, 10, 60):
            v, i = _local_topk(S, lo, hi, k, lambda b, j: j)
            ti = torch.from_numpy(i)
            gi, gv = all_gather_topk(torch.from_numpy(v), ti, ordinal_tiebreak(ti), k)
            for b in range(B):
                ref = np.lexsort((np.arange(N), -S[b]))[:k]
                ok.append(gi[b].tolist() == ref.tolist())
                ok.append(np.array_equal(gv[b].numpy(), S[b, ref]))
        # (2) final ranking: own entry first, then id rank (index.py:290-294)
        for k in (3, 10, 103):
            def tbf(b, j):
                return 0 if j == self_global[b] else 1 + idrank[j]
            v, i = _local_topk(S, lo, hi, k, tbf)
            ti = torch.from_numpy(i)
            tb = ranking_tiebreak(ti, torch.from_numpy(idrank), torch.from_numpy(self_global))
            gi, gv = all_gather_topk(torch.from_numpy(v), ti, tb, k)
            for b in range(B):
                not_self = np.arange(N) != self_global[b]
                ref = np.lexsort((idrank, not_self, -S[b]))[:k]
                ok.append(gi[b].tolist() == ref.tolist())
        results[rank] = all(ok)
    finally:
        dist.destroy_process_group()


def test_sharded_topk_merge_world2_gloo():
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(2, port, results), nprocs=2, join=True,
                       start_method="spawn")
    assert dict(results) == {0: True, 1: True}


@pytest.mark.parametrize("n,world", [(10, 3), (7, 8), (1000, 8), (5, 1)])
def test_shard_bounds_partition(n, world):
    cover = []
    for r in range(world):
        lo, hi = shard_bounds(n, world, r)
        assert 0 <= lo <= hi <= n
        assert hi - lo in (n // world, n // world + 1)
        cover.extend(range(lo, hi))
    assert cover == list(range(n))


def test_pack_round_trip_and_missing_entries():
    vals = torch.tensor([[0.5, 0.0, 1e-300, -2.5]], dtype=torch.float64)
    idx = torch.tensor([[3, -1, 2**31 - 1, 0]])
    tb = torch.tensor([[3, 7, 0xFFFFFFFE, 0]])
    v, o, t = unpack_candidates(pack_candidates(vals, idx, tb))
    assert torch.equal(v, vals)
    assert o.tolist() == [[3, -1, 2**31 - 1, 0]]
    assert (t.to(torch.int64) & 0xFFFFFFFF).tolist() == [[3, 0xFFFFFFFF, 0xFFFFFFFE, 0]]
    i, val = host_merge(v, o, t, 3, False)
    assert i.tolist() == [[3, 2**31 - 1, 0]]
