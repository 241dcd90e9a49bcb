"""Shard-by-shape path on the GPU: build_sharded + ShardedEngine at world
size 1 and 2 must rank exactly like the single-GPU engine.  World size 2 runs
two processes on the one available GPU with gloo collectives (host-side
exchanges; no kernel waits on another rank)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cases import E2E_CASES, mixture_views, sampled_codebook, shape_ids

pytestmark = pytest.mark.gpu


def _case(i):
    if i == "fp16":  # fp16 storage, cells probed >= 192 times: the dense-cell scan
        views, _ = mixture_views(83, 600, 8, 64, 5, n_queries=100)
        db = views[:600].astype(np.float16)
        qs = views[600:].astype(np.float16).astype(np.float32)
        C = sampled_codebook(db.astype(np.float32), 3, 4)
        return db, qs, C, dict(n_views=8, codebook_size=3, ma=1, k1=6, k2=3, imported=True,
                               storage_dtype="float16", similarity="gaussian"), 20
    name, seed, N, V, d, classes, K, ma, k1, k2, nq, top_k, zv = E2E_CASES[i]
    views, _ = mixture_views(seed, N, V, d, classes, zero_views=zv, n_queries=nq)
    C = sampled_codebook(views[:N], K, seed + 1)
    return views[:N], views[N:], C, dict(n_views=V, codebook_size=K, ma=ma, k1=k1, k2=k2,
                                          imported=True), top_k


def _single(db, qs, C, cfgkw, top_k):
    import paper_1604_01879_b200 as gift
    from paper_1604_01879_b200.codebook import Codebook

    cfg = gift.IndexConfig(**cfgkw)
    b = gift.build_index_from_views(db, shape_ids(len(db)), cfg,
                                    codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")})
    Q = torch.from_numpy(qs).cuda()
    i, v = b.engine.run(Q, top_k=top_k, rerank=True)
    return i.cpu().numpy().astype(np.int64), v.cpu().numpy()


def _sharded(rank, world, db, qs, C, cfgkw, top_k):
    from paper_1604_01879_b200 import IndexConfig
    from paper_1604_01879_b200 import engine as eg
    from paper_1604_01879_b200.dist import ShardedEngine, build_sharded, shard_bounds

    cfg = IndexConfig(**cfgkw)
    N = len(db)
    lo, hi = shard_bounds(N, world, rank)
    X = torch.from_numpy(np.ascontiguousarray(db[lo:hi])).cuda()
    fif, raw, sif = build_sharded(X, eg.DeviceCodebook.from_numpy(C), cfg, N)
    idrank = torch.arange(N, dtype=torch.int32, device="cuda")  # zero-padded ids: rank == ordinal
    eng = ShardedEngine(fif, raw, sif, idrank, cfg, N)
    Q = torch.from_numpy(qs).cuda()
    i, v = eng.run(Q, top_k, rerank=True)
    # batches in flight on two streams give the same rankings
    half = (Q.shape[0] + 1) // 2
    outs = eng.run_many([Q[:half].contiguous(), Q[half:].contiguous()], top_k, lanes=2)
    torch.cuda.synchronize()
    i2 = torch.cat([o[0] for o in outs]).cpu().numpy()
    v2 = torch.cat([o[1] for o in outs]).cpu().numpy()
    np.testing.assert_array_equal(i2, i.cpu().numpy())
    np.testing.assert_array_equal(v2, v.cpu().numpy())
    return i.cpu().numpy().astype(np.int64), v.cpu().numpy()


def _worker(rank, world, port, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        db, qs, C, cfgkw, top_k = _case(case)
        i, v = _sharded(rank, world, db, qs, C, cfgkw, top_k)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), i=i, v=v)
    finally:
        dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case", [1, 2, "fp16"])
def test_sharded_world1_equals_single(case):
    db, qs, C, cfgkw, top_k = _case(case)
    ref_i, ref_v = _single(db, qs, C, cfgkw, top_k)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        i, v = _sharded(0, 1, db, qs, C, cfgkw, top_k)
    finally:
        dist.destroy_process_group()
    np.testing.assert_array_equal(i, ref_i)
    np.testing.assert_array_equal(v, ref_v)


@pytest.mark.parametrize("case", [1, 2, "fp16"])
def test_sharded_world2_equals_single(case):
    db, qs, C, cfgkw, top_k = _case(case)
    ref_i, ref_v = _single(db, qs, C, cfgkw, top_k)
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(_worker, args=(2, _port(), case, td), nprocs=2, join=True,
                           start_method="spawn")
        for r in range(2):
            got = np.load(os.path.join(td, f"r{r}.npz"))
            np.testing.assert_array_equal(got["i"], ref_i)
            np.testing.assert_array_equal(got["v"], ref_v)
