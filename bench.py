"""Benchmark of the GIFT F-IF + S-IF query path (BASELINE.json metric:
queries/sec, F-IF match + S-IF re-rank; F-IF scan HBM GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gift|reference]
                    [--config c2]

A step = one batch of queries (config 2: 64 queries x 64 views x d=4096)
through quantize -> F-IF scan -> top-k2 -> query activation -> S-IF ->
top-100, against a 10,000-shape database resident in HBM.  `value` is
device-timed (CUDA events, inputs resident); `e2e` runs the public API
`query_many` from pinned host memory (H2D of every batch and D2H of its
results inside the timed region).  Under torchrun (N > 1) every rank serves
an index replica and a disjoint query stream ("replicas": the 10 GB
database of config 2 fits one GPU; sharding is for configs 3-5).

--impl reference times the reference's CPU path (oracle/ numpy port of
shapesearch's query_fif + rerank_scores, single-channel variant) on all host
cores; its index lists come from the parity-verified GPU build (the CPU
build of config 2 would take hours).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1604_01879_b200 import IndexConfig, build_index_from_views, query_many  # noqa: E402
from paper_1604_01879_b200.index import LANE_RESERVE_SMS, lane_streams  # noqa: E402
from paper_1604_01879_b200 import engine as eg  # noqa: E402
from paper_1604_01879_b200 import synth  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402

METRIC = "queries/sec (F-IF match + S-IF rerank)"
UNIT = "queries/s"
SEED = 20160407


# ------------------------------------------------------------------ helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, period_ms: int = 200):
        self.gpu = gpu
        self.period_ms = period_ms
        self.proc = None
        self.lines = []

    def __enter__(self):
        if os.environ.get("GIFT_BENCH_NO_SMI") == "1":  # diagnostics: no sampler
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms",
                 os.environ.get("GIFT_SMI_MS", str(self.period_ms))],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        # nvidia-smi's start-up (NVML init) stalls the GPU for tens of ms:
        # wait for its first samples before the caller's timed region starts
        t0 = time.time()
        while self.proc is not None and len(self.lines) < 2 and time.time() - t0 < 15.0:
            time.sleep(0.05)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


# (batches in flight, SMs the scan leaves to the other lanes) per config:
# config 2's non-scan kernels are ~20% of a step and overlap the next
# batches' scans; config 3 (owner reduce, 105 GB) and config 4 (tensor-bound
# scan) measured no gain
DEFAULT_LANES = {"c1": (4, LANE_RESERVE_SMS), "c2": (4, LANE_RESERVE_SMS)}


def warm(fn, iters: int, min_s: float = 0.25):
    """Untimed warm-up: at least `iters` calls and `min_s` seconds of
    back-to-back GPU work, ending with a synchronize.  Runs inside the clock
    sampler so the timed region starts on a busy GPU (a GPU left idle while
    the sampler starts loses ~30 ms to the clock ramp on latency-bound steps)."""
    t0 = time.time()
    i = 0
    while i < iters or time.time() - t0 < min_s:
        fn(i)
        i += 1
        if i >= iters:
            torch.cuda.synchronize()
    torch.cuda.synchronize()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def count_launches(fn) -> int:
    """Kernels of libgift.so one call of fn launches (CUPTI via torch.profiler,
    names in namespace gift::), measured outside the timed region."""
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return sum(1 for e in prof.events()
               if e.device_type.name == "CUDA" and "gift::" in e.name)


def measured_tensor_peak():
    """Dense bf16/fp16 tensor peak (TFLOP/s): MEASURED_PEAKS.json burst figure
    (the scan is timed per launch), else the profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return 1590.0


def scan_work(eng, Q, w, top_k):
    """Algorithmic bytes / flops of one scan launch:
    bytes = sum_{c in U} |c| (d s_feat + 4 [+4 |p|^2]) + B V d 4 + B k 8,
    flops = sum_c M_c |c| 2 d."""
    fif = eng.fa
    B, V, d = Q.shape
    flat = Q.reshape(-1, d)
    nz, _ = eg.view_prep(flat)
    cells = eg.quantize_rows(fif.cb, flat, w.ma, nz=nz).reshape(-1)
    cells = cells[cells >= 0].long()
    counts = torch.bincount(cells, minlength=fif.cb.K).double()
    sizes = (fif.cell_off[1:] - fif.cell_off[:-1]).double()
    s_feat = 2 if w.storage == "float16" else 4
    per_post = d * s_feat + 4 + (4 if eng.cfg.similarity == "gaussian" else 0)
    used = counts > 0
    nbytes = float((sizes[used] * per_post).sum()) + B * V * d * 4 + B * top_k * 8
    flops = float((counts * sizes).sum()) * 2 * d
    return nbytes, flops


def load_ncu(config):
    """ncu --set full summary of this workload's scan / quantizer launch
    (profiles/ncu_summary.json, captured on one timed-path batch)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config) or {}
    except (OSError, ValueError):
        return {}


def load_traffic(config):
    n = load_ncu(config)
    if "scan_dram_read_bytes" not in n:
        return None
    return n["scan_dram_read_bytes"] + n.get("scan_dram_write_bytes", 0)


# ------------------------------------------------------------------ setup
def build_streamed(w, device):
    """Config 3: 105 GB of f32 views on one GPU.  The database is generated
    block by block on the device and streamed through the chunked build
    (quantize pass, scatter into the tensor-core planes, self-join); the index
    keeps only the planes (52 GB hi + 52 GB lo)."""
    from paper_1604_01879_b200 import build_index_streamed

    mix = synth.BlockMixture(w, SEED, device)
    C = synth.sample_centroids_rows(mix, w.K, SEED + 1).cpu().numpy()
    qs = mix.queries()
    cfg = IndexConfig(n_views=w.n_views, codebook_size=w.K, ma=w.ma, k1=w.k1, k2=w.k2,
                      similarity="gaussian", sigma=w.sigma, storage_dtype=w.storage,
                      batch_size=w.batch, imported=True)
    t0 = time.perf_counter()
    bundle = build_index_streamed(mix.provider(), synth.shape_ids(w.n_shapes), w.n_views, w.dim,
                                  cfg, codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")},
                                  chunk=1024, keep_features=False, self_join_batch=w.batch)
    torch.cuda.synchronize()
    return bundle, qs, time.perf_counter() - t0


def build(w, device):
    if w.name == "c3":
        return build_streamed(w, device)
    if w.storage == "float16":  # config 4: Zipf-skewed cells, fp16 storage
        db, qs, Ct = synth.zipf_mixture(w, SEED, device)
        C = Ct.cpu().numpy()
    else:
        db, qs, _labels = synth.mixture(w, SEED, device)
        C = synth.sample_centroids(db, w.K, SEED + 1).cpu().numpy()
    cfg = IndexConfig(n_views=w.n_views, codebook_size=w.K, ma=w.ma, k1=w.k1, k2=w.k2,
                      similarity="gaussian", sigma=w.sigma, storage_dtype=w.storage,
                      batch_size=w.batch, imported=True)
    ids = synth.shape_ids(w.n_shapes)
    t0 = time.perf_counter()
    bundle = build_index_from_views(db, ids, cfg, codebooks={"A": Codebook(C, "A"),
                                                             "B": Codebook(C, "B")})
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    del db
    torch.cuda.empty_cache()
    return bundle, qs, build_s


def host_oracle(bundle, w):
    """oracle.OracleIndex over the (parity-verified) GPU-built lists."""
    import oracle

    fif = bundle.fifs["A"]
    ords, feats = fif.entry_ordinals, fif.entry_features
    raw = [oracle.Act(a.indices, a.values, a.norm) for a in bundle.raw_activations["A"]]
    sif = oracle.Sif(norms=bundle.sif.norms, entry_ordinals=bundle.sif.entry_ordinals,
                     entry_values=bundle.sif.entry_values)
    orc = oracle.OracleIndex.from_parts(
        bundle.shape_ids, fif.codebook.centroids, ords, feats, raw, sif, ma=w.ma, k1=w.k1,
        k2=w.k2, alpha=0.5, similarity="gaussian_expanded", sigma=w.sigma)
    for e in range(len(ords)):  # |p|^2 per cell, computed once before forking
        orc.fifs["A"].pnorm2(e)
    return orc


_ORACLE = None
_QUERIES = None


def _cpu_query(i):
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        res, _ = _ORACLE.query(_QUERIES[i], top_k=100, rerank=True)
    return len(res)


def cpu_sample(orc, queries_host, n_procs, n_queries):
    """Wall time of n_queries oracle queries on n_procs forked workers."""
    import multiprocessing as mp

    global _ORACLE, _QUERIES
    _ORACLE, _QUERIES = orc, queries_host
    ctx = mp.get_context("fork")
    with ctx.Pool(n_procs) as pool:
        pool.map(_cpu_query, [0] * min(n_procs, 2))  # warm the forked workers
        t0 = time.perf_counter()
        pool.map(_cpu_query, [i % len(queries_host) for i in range(n_queries)], chunksize=1)
        return time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ arms
def run_reference(args, w):
    ws, rank, local = dist_env()
    if ws > 1 and rank != 0:
        return
    torch.cuda.set_device(local)
    bundle, qs, _ = build(w, torch.device("cuda", local))  # setup only (not timed)
    orc = host_oracle(bundle, w)
    qh = qs[: max(64, w.batch)].cpu().numpy()
    del bundle
    torch.cuda.empty_cache()
    cores = host_cores()
    per_step = cores  # one query per worker per step
    for _ in range(args.warmup):
        cpu_sample(orc, qh, cores, min(cores, 4))
    times = [cpu_sample(orc, qh, cores, per_step) for _ in range(args.steps)]
    qps = per_step * len(times) / sum(times)
    sample = (f"{per_step} queries/step x {len(times)} steps of config {w.name} "
              f"(single-channel oracle port of query_fif+rerank_scores, gaussian via GEMV)")
    line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n_shapes": w.n_shapes, "n_views": w.n_views,
                       "dim": w.dim, "K": w.K, "ma": w.ma, "sigma": w.sigma, "top_k": w.top_k},
            "cpu_baseline": {"value": qps, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": qps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_c5(args):
    """Config 5 (re-rank dominated): given top-50 lists for 1M shapes, S-IF
    over all shapes, queries re-ranked with k = 50 neighbour-set Jaccard."""
    from paper_1604_01879_b200 import build_index_from_lists

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    c = synth.C5
    n = args.c5_shapes or c["n_shapes"]
    idx, val = synth.community_lists(SEED, device, n_shapes=n)
    cfg = IndexConfig(k1=c["list_len"], k2=c["k2"], imported=True, batch_size=c["batch"])
    t0 = time.perf_counter()
    bundle = build_index_from_lists(idx, val, synth.shape_ids(n), cfg)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    eng = bundle.engine
    g = torch.Generator(device=device)
    g.manual_seed(SEED + 5)
    B = c["batch"]
    qrows = torch.randint(0, n, (B * (args.steps + args.warmup),), generator=g, device=device)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def step(i):
        r = qrows[(i % args.warmup) * B:(i % args.warmup + 1) * B]
        eng.rerank_lists(idx[r], val[r], top_k=c["top_k"], self_local=r.to(torch.int32))

    with ClockSampler(local) as clk:
        warm(step, args.warmup)
        ev[0].record()
        for i in range(args.warmup, args.warmup + args.steps):
            r = qrows[i * B:(i + 1) * B]
            eng.rerank_lists(idx[r], val[r], top_k=c["top_k"], self_local=r.to(torch.int32))
        ev[1].record()
        torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    per_step = count_launches(lambda: step(0))
    line = {"metric": METRIC, "value": B * args.steps / (ms / 1000), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "c5", "n_shapes": n, "list_len": c["list_len"],
                       "communities": c["communities"], "k2": c["k2"], "top_k": c["top_k"],
                       "batch": B, "sif_postings": int(bundle.sif.dev.e_ord.numel()),
                       "build_s": build_s},
            "e2e": None, "gpu_launches": per_step * args.steps, "roofline": None,
            "cpu_baseline": None,
            "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_sharded(args, w):
    """Database sharded by shape over the ranks (dist.py): every rank holds
    N / G shapes (all cells), queries are replicated, per-shard top-k2 and
    top-k candidates are merged with NCCL all_gather_into_tensor."""
    from paper_1604_01879_b200 import engine as eg2
    from paper_1604_01879_b200.dist import ShardedEngine, build_sharded, shard_bounds

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=device)
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo", rank=0, world_size=1)
    if w.storage == "float16":
        db, qs, Ct = synth.zipf_mixture(w, SEED, device)
        C = Ct.cpu().numpy()
    else:
        db, qs, _ = synth.mixture(w, SEED, device)
        C = synth.sample_centroids(db, w.K, SEED + 1).cpu().numpy()
    lo, hi = shard_bounds(w.n_shapes, ws, rank)
    X = db[lo:hi].contiguous()
    del db
    torch.cuda.empty_cache()
    cfg = IndexConfig(n_views=w.n_views, codebook_size=w.K, ma=w.ma, k1=w.k1, k2=w.k2,
                      similarity="gaussian", sigma=w.sigma, storage_dtype=w.storage,
                      batch_size=w.batch, imported=True)
    t0 = time.perf_counter()
    fif, raw, sif = build_sharded(X, eg2.DeviceCodebook.from_numpy(C), cfg, w.n_shapes)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    del X
    idrank = torch.arange(w.n_shapes, dtype=torch.int32, device=device)  # zero-padded ids
    eng = ShardedEngine(fif, raw, sif, idrank, cfg, w.n_shapes)
    B = w.batch
    nb = max(1, qs.shape[0] // B)
    batches = [qs[j * B:(j + 1) * B].contiguous() for j in range(nb)]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with ClockSampler(local) as clk:
        warm(lambda i: eng.run(batches[i % nb], w.top_k), args.warmup)
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        for i in range(args.steps):
            eng.run(batches[(args.warmup + i) % nb], w.top_k)
        ev[1].record()
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([ev[0].elapsed_time(ev[1])], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        line = {"metric": METRIC, "value": B * args.steps / (ms / 1000.0), "unit": UNIT,
                "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": w.name, "n_shapes": w.n_shapes, "parallelism":
                           f"shard{ws}", "batch": B, "top_k": w.top_k, "build_s": build_s},
                "e2e": None, "gpu_launches": None, "roofline": None, "cpu_baseline": None,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_gift(args, w):
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=device)
    bundle, qs, build_s = build(w, device)
    eng = bundle.engine
    B = w.batch
    nb = max(1, qs.shape[0] // B)
    order = [(rank + i * ws) % nb for i in range(args.steps + args.warmup)]
    batches = [qs[j * B:(j + 1) * B].contiguous() for j in range(nb)]
    stream = torch.cuda.current_stream()
    # batch i runs on lane i % L: its own stream and scratch, so one batch's
    # quantize / reduce / re-rank kernels overlap the other batch's scan
    lanes_default, reserve_default = DEFAULT_LANES.get(w.name, (1, 0))
    L = max(1, args.lanes if args.lanes is not None else lanes_default)
    lanes = [stream] if L == 1 else lane_streams(L)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    scan_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    for i, (a, b) in enumerate(scan_ev):  # torch creates CUDA events lazily, on first record
        a.record(lanes[i % L])
        b.record(lanes[i % L])

    # SMs the scan leaves to the other lanes' kernels (DEFAULT_LANES)
    if args.reserve_sms is not None:
        eng.reserve_sms = args.reserve_sms
    else:
        eng.reserve_sms = reserve_default if L > 1 else 0

    def step(i, bi, sev=None):
        s = lanes[i % L]
        with torch.cuda.stream(s):
            eng.run(batches[bi], top_k=w.top_k, rerank=True, scan_events=sev)

    with ClockSampler(local) as clk:
        for s in lanes:
            s.wait_stream(stream)
        warm(lambda i: step(i, order[i % args.warmup]), max(args.warmup, L))
        for s in lanes:
            stream.wait_stream(s)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        for s in lanes:
            s.wait_event(ev[0])
        for i in range(args.steps):
            step(i, order[args.warmup + i], scan_ev[i])
        for s in lanes:
            stream.wait_stream(s)
        ev[1].record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        # the scan's own duration: with batches in flight a scan's events also
        # span its wait behind the previous batch's scan, so the kernel time
        # for the roofline comes from the same batches run one at a time
        # right after (CUDA events on the launching stream, inside the sampler)
        if L > 1:
            reserve, eng.reserve_sms = eng.reserve_sms, 0
            serial_ev = [(torch.cuda.Event(enable_timing=True),
                          torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for a, b in serial_ev:
                a.record(stream)
                b.record(stream)
            torch.cuda.synchronize()
            for i in range(args.steps):
                eng.run(batches[order[args.warmup + i]], top_k=w.top_k, rerank=True,
                        scan_events=serial_ev[i])
            torch.cuda.synchronize()
            eng.reserve_sms = reserve
        else:
            serial_ev = scan_ev
    ms = ev[0].elapsed_time(ev[1])
    launches_per_step = count_launches(
        lambda: eng.run(batches[order[args.warmup]], top_k=w.top_k, rerank=True))
    scan_ms = [a.elapsed_time(b) for a, b in serial_ev]
    scan_ms_overlapped = [a.elapsed_time(b) for a, b in scan_ev]
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_q = B * args.steps * ws
    value = total_q / (ms_max / 1000.0)

    # ---- e2e through the public API from pinned host memory
    host = torch.empty((args.steps * B, w.n_views, w.dim), dtype=torch.float32, pin_memory=True)
    for i in range(args.steps):
        host[i * B:(i + 1) * B].copy_(batches[order[args.warmup + i]])
    query_many(bundle, host[:L * B], top_k=w.top_k, lanes=L,
               reserve_sms=eng.reserve_sms)  # warm
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    query_many(bundle, host, top_k=w.top_k, lanes=L, reserve_sms=eng.reserve_sms)
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = total_q / float(t.item())

    # ---- roofline of the dominant kernel (F-IF scan)
    work = [scan_work(eng, batches[order[args.warmup + i]], w, w.top_k) for i in range(args.steps)]
    nbytes = sum(x[0] for x in work) / len(work)
    flops = sum(x[1] for x in work) / len(work)
    scan_avg_ms = sum(scan_ms) / len(scan_ms)
    peak, peak_kind = measured_peaks()
    tpeak = measured_tensor_peak()
    scan_s = scan_avg_ms / 1000.0
    achieved = nbytes / scan_s / 1e9
    achieved_tf = flops / scan_s / 1e12
    # roofline: the slower of the HBM time and the tensor time of the
    # algorithmic work; the fp32 split runs 2 (fp16 storage)
    # or 3 (f32) fp16 MMA products per algorithmic product on the tensor cores
    t_hbm = nbytes / (peak * 1e9)
    t_tc = flops / (tpeak * 1e12)
    split = 2 if w.storage == "float16" else 3
    if t_tc > t_hbm:
        roofline = {"bound": "tensor", "achieved": achieved_tf, "peak": tpeak, "unit": "TFLOP/s",
                    "frac": achieved_tf / tpeak}
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak}
    roofline.update({"kernel": "fif_scan_tc_kernel", "peak_source": peak_kind,
                     "traffic": load_traffic(w.name), "alg_bytes_per_launch": nbytes,
                     "alg_flops_per_launch": flops, "scan_ms_avg": scan_avg_ms,
                     "scan_ms_measured": ("serial pass over the timed batches" if L > 1
                                          else "timed region"),
                     "scan_ms_avg_in_flight": sum(scan_ms_overlapped) / len(scan_ms_overlapped),
                     "scan_share_of_step": scan_avg_ms * args.steps / ms,
                     "achieved_gbs": achieved, "hbm_frac": achieved / peak,
                     "achieved_tflops": achieved_tf, "tensor_frac": achieved_tf / tpeak,
                     "fp16_mma_products_per_alg_product": split,
                     "tensor_pipe_frac_incl_split": achieved_tf * split / tpeak})
    ncu = load_ncu(w.name)
    quant_ncu = ({"kernel": ncu["quantize_kernel"], "tensor_hmma_active_pct":
                  ncu["quantize_tensor_hmma_active_pct"], "source": "ncu --set full"}
                 if "quantize_kernel" in ncu else None)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and eng.fa.feat is not None:
        orc = host_oracle(bundle, w)
        qh = batches[0].cpu().numpy()
        cores = host_cores()
        n = cores
        wall = cpu_sample(orc, qh, cores, n)
        cpu = {"value": n / wall, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{n} config-{w.name} queries on {cores} forked workers "
                         f"(oracle port of query_fif+rerank_scores, single channel)"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": w.name, "n_shapes": w.n_shapes, "n_views": w.n_views,
                           "dim": w.dim, "K": w.K, "ma": w.ma, "similarity": "gaussian",
                           "sigma": w.sigma, "k1": w.k1, "k2": w.k2, "top_k": w.top_k,
                           "batch": B, "parallelism": f"replicas{ws}",
                           "lanes": L, "scan_reserved_sms": eng.reserve_sms,
                           "storage": w.storage, "n_queries": w.n_queries,
                           "l2": "inputs larger than L2 (database >= 10.5 GB)",
                           "features": "planes only (streamed build)" if eng.fa.feat is None
                           else "storage copy + planes",
                           "build_s": build_s},
                "e2e": {"value": e2e_value, "unit": UNIT,
                        "h2d_bytes_per_step": B * w.n_views * w.dim * 4,
                        "d2h_bytes_per_step": B * w.top_k * 12},
                "gpu_launches": launches_per_step * args.steps,
                "roofline": roofline, "quantize": quant_ncu, "cpu_baseline": cpu,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gift", choices=["gift", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(synth.WORKLOADS) + ["c5"])
    ap.add_argument("--c5-shapes", type=int, default=0, help="override config-5 N (smoke runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reserve-sms", type=int, default=None,
                    help="SMs the scan leaves to other lanes (default per config, "
                         "DEFAULT_LANES)")
    ap.add_argument("--lanes", type=int, default=None,
                    help="batches in flight on separate streams (1 = serial; default "
                         "per config, DEFAULT_LANES)")
    ap.add_argument("--shard", action="store_true",
                    help="shard the database by shape over the ranks (configs 3/4)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "gift" else args.warmup
    if args.config == "c5":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 5 reference arm not "
                              "provided (oracle S-IF build of 1M shapes takes hours)"}))
            return
        run_c5(args)
        return
    w = synth.WORKLOADS[args.config]
    if args.impl == "reference":
        run_reference(args, w)
    elif args.shard:
        run_sharded(args, w)
    else:
        run_gift(args, w)


if __name__ == "__main__":
    main()
