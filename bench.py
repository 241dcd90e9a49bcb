"""Benchmark of the GIFT F-IF + S-IF query path (BASELINE.json metric:
queries/sec, F-IF match + S-IF re-rank; F-IF scan HBM GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gift|reference]
                    [--config c1|c2|c3|c4|c5|...] [--shard]

A step = one batch of queries (config 2: 64 queries x 64 views x d=4096)
through quantize -> F-IF scan -> top-k2 -> query activation -> S-IF ->
top-100, against a 10,000-shape database resident in HBM.  `value` is
device-timed (CUDA events, inputs resident); `e2e` runs the public API
(`query_many`, or the sharded engine) from pinned host memory, the H2D copy
of every batch and the D2H of its results inside the timed region.

--gpus N: under torchrun WORLD_SIZE must equal N; without torchrun, N > 1
re-launches this script with `torch.distributed.run` (one rank per GPU).
At N > 1 configs 1-2 serve one index replica per rank (the database fits
one GPU; disjoint query streams, no collective), configs 3-5 shard the
database by shape (dist.py: two packed all-gathers per batch).

--impl reference times the reference's own CPU path (the oracle/ port of
shapesearch's query_fif + rerank_scores + ranking) on all host cores, over
an index the ORACLE builds on the host (bit-exact quantize, f64 self-join):
this arm never imports the product package nor maps libgift.so.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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

METRIC = "queries/sec (F-IF match + S-IF rerank)"
UNIT = "queries/s"
SEED = 20160407


def _load_synth():
    """The workload generators (paper_1604_01879_b200/synth.py, torch only),
    loaded by path: the reference arm must not import the product package
    (nor map libgift.so)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "gift_workloads", os.path.join(ROOT, "paper_1604_01879_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["gift_workloads"] = mod  # dataclasses resolve their module by name
    spec.loader.exec_module(mod)
    return mod


synth = _load_synth()


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
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
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


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def measured_peaks():
    p = _peaks()
    if "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def measured_tensor_peak():
    """Dense bf16/fp16 tensor peak (TFLOP/s): MEASURED_PEAKS.json burst figure
    (the scan is timed per launch), else the profiling recipe's fallback."""
    return float(_peaks().get("bf16_tflops", 1590.0))


_SYNC_APIS = ("cudaStreamSynchronize", "cudaDeviceSynchronize", "cudaEventSynchronize",
              "cudaMemcpy", "cudaMemcpy2D", "cudaMemset")  # host-blocking runtime calls


def count_launches(fn, syncs: dict | None = None) -> int:
    """Kernels of libgift.so one call of fn launches (CUPTI via torch.profiler,
    names in namespace gift::), measured outside the timed region; with
    `syncs`, also counts the host-blocking CUDA runtime calls fn makes (the
    query path should make none)."""
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        fn()
    evs = prof.events()
    if syncs is not None:
        for e in evs:
            if e.device_type.name == "CPU" and e.name in _SYNC_APIS:
                syncs[e.name] = syncs.get(e.name, 0) + 1
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as base:
            pass  # the profiler's own calls (its stop synchronizes the device)
        for e in base.events():
            if e.device_type.name == "CPU" and e.name in syncs:
                syncs[e.name] -= 1
        for k in [k for k, v in syncs.items() if v <= 0]:
            del syncs[k]
    torch.cuda.synchronize()
    return sum(1 for e in evs if e.device_type.name == "CUDA" and "gift::" in e.name)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def host_info():
    """CPU model, cores and RAM of the host the CPU baseline runs on."""
    model, phys = None, set()
    try:
        with open("/proc/cpuinfo") as fh:
            cur = {}
            for line in fh:
                if ":" in line:
                    k, v = (x.strip() for x in line.split(":", 1))
                    cur[k] = v
                    if k == "model name":
                        model = v
                elif cur:
                    phys.add((cur.get("physical id"), cur.get("core id")))
                    cur = {}
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemTotal:"):
                    ram = round(int(line.split()[1]) / 2**20, 1)
    except OSError:
        pass
    return {"cpu_model": model, "physical_cores": len(phys) or None,
            "threads_available": host_cores(), "ram_gib": ram}


def workload_config(w, parallelism: str) -> dict:
    """The workload keys both arms report (the driver compares them)."""
    return {"workload": w.name, "n_shapes": w.n_shapes, "n_views": w.n_views, "dim": w.dim,
            "K": w.K, "ma": w.ma, "similarity": "gaussian", "sigma": w.sigma, "k1": w.k1,
            "k2": w.k2, "top_k": w.top_k, "batch": w.batch, "n_queries": w.n_queries,
            "storage": w.storage, "parallelism": parallelism,
            "l2": "inputs larger than L2 (database >= 65 MB per GPU, batch inputs streamed)"}


def c5_communities(n):
    return synth.C5["communities"] if n >= synth.C5["n_shapes"] else max(1, n // 500)


def c5_config(c, n, parallelism):
    return {"workload": "c5", "n_shapes": n, "list_len": c["list_len"],
            "communities": c5_communities(n), "k1": c["list_len"], "k2": c["k2"],
            "top_k": c["top_k"], "batch": c["batch"], "n_queries": c["n_queries"],
            "parallelism": parallelism,
            "l2": "inputs larger than L2 (S-IF of 1M shapes ~2.2 GB)"}


# ------------------------------------------------------------------ GPU arm
GRAPH_CONFIGS = ("c1",)  # configs whose timed batches replay CUDA graphs by default


def default_lanes(name):
    """(batches in flight, SMs the scan leaves to the other lanes) per config:
    config 2's non-scan kernels are ~20% of a step and overlap the next
    batches' scans (profiles/r02/c2_lanes_reserve_sweep.json); configs 3 and 4
    (no host synchronisation left in the query path) gain 3% / 2% from two
    lanes with 20 SMs left to the other lane; config 1 replays CUDA graphs and
    saturates at 6-8 lanes (profiles/r02/c1_graph_lanes_s4/: 4 lanes 890k,
    8 lanes 1.01M q/s)."""
    from paper_1604_01879_b200.index import LANE_RESERVE_SMS

    return {"c1": (8, LANE_RESERVE_SMS), "c2": (4, LANE_RESERVE_SMS),
            "c3": (2, 20), "c4": (2, 20)}.get(name, (1, 0))


def scan_work(fif, Q, w, top_k, similarity="gaussian"):
    """Algorithmic bytes / flops of one scan launch:
    bytes = sum_{c in U} |c| (d s_feat + 4 [+4 |p|^2]) + B V d 4 + B k 8,
    flops = sum_c M_c |c| 2 d."""
    from paper_1604_01879_b200 import engine as eg

    B, V, d = Q.shape
    flat = Q.reshape(-1, d)
    nz, _ = eg.view_prep(flat)
    cells = eg.quantize_rows(fif.cb, flat, w.ma, nz=nz).reshape(-1)
    cells = cells[cells >= 0].long()
    counts = torch.bincount(cells, minlength=fif.cb.K).double()
    sizes = (fif.cell_off[1:] - fif.cell_off[:-1]).double()
    s_feat = 2 if w.storage == "float16" else 4
    per_post = d * s_feat + 4 + (4 if similarity == "gaussian" else 0)
    used = counts > 0
    nbytes = float((sizes[used] * per_post).sum()) + B * V * d * 4 + B * top_k * 8
    flops = float((counts * sizes).sum()) * 2 * d
    return nbytes, flops


def load_ncu(config):
    """ncu --set full summary of this workload's scan / quantizer launch
    (profiles/ncu_summary.json, captured on one timed-path batch)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            return json.load(fh).get(config) or {}
    except (OSError, ValueError):
        return {}


def load_traffic(config):
    n = load_ncu(config)
    if "scan_dram_read_bytes" not in n:
        return None
    return n["scan_dram_read_bytes"] + n.get("scan_dram_write_bytes", 0)


def scan_kernel_name(w, what=""):
    """The scan's kernels: fp16 storage runs the dense cells (>= 192 probes
    per batch) on fif_scan_dense_kernel and the others on fif_scan_tc_kernel,
    one after the other on the stream, both inside the scan events."""
    k = ("fif_scan_dense_kernel + fif_scan_tc_kernel (dense / other cells)"
         if w.storage == "float16" else "fif_scan_tc_kernel")
    return k + what


def fp16_exact(batches):
    """Every query value exactly an fp16 (config 4's fp16-rounded views): the
    scan then drops the query lo plane (one fp16 MMA product per product)."""
    return all(bool((b.to(torch.float16).to(b.dtype) == b).all()) for b in batches)


def roofline_of(nbytes, flops, scan_ms, w, kernel, measured, q16=False):
    """The slower of the HBM time and the tensor time of the algorithmic
    work; the fp32 split runs 3 (f32 planes), 2 (fp16
    storage) or 1 (fp16 storage, fp16-exact queries) fp16 MMA products per
    algorithmic product on the tensor cores."""
    peak, peak_kind = measured_peaks()
    tpeak = measured_tensor_peak()
    scan_s = scan_ms / 1000.0
    achieved = nbytes / scan_s / 1e9
    achieved_tf = flops / scan_s / 1e12
    t_hbm = nbytes / (peak * 1e9)
    t_tc = flops / (tpeak * 1e12)
    split = (1 if q16 else 2) if w.storage == "float16" else 3
    if t_tc > t_hbm:
        r = {"bound": "tensor", "achieved": achieved_tf, "peak": tpeak, "unit": "TFLOP/s",
             "frac": achieved_tf / tpeak}
    else:
        r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
             "frac": achieved / peak}
    r.update({"kernel": kernel, "peak_source": peak_kind, "traffic": load_traffic(w.name),
              "alg_bytes_per_launch": nbytes, "alg_flops_per_launch": flops,
              "scan_ms_avg": scan_ms, "scan_ms_measured": measured,
              "achieved_gbs": achieved, "hbm_frac": achieved / peak,
              "achieved_tflops": achieved_tf, "tensor_frac": achieved_tf / tpeak,
              "fp16_mma_products_per_alg_product": split})
    return r


def build_streamed(w, device):
    """Config 3: 105 GB of f32 views on one GPU.  The database is generated
    block by block on the device and streamed through the chunked build
    (quantize pass, scatter into the tensor-core planes, self-join); the index
    keeps only the planes (52 GB hi + 52 GB lo)."""
    from paper_1604_01879_b200 import IndexConfig, build_index_streamed
    from paper_1604_01879_b200.codebook import Codebook

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


def generate(w, device):
    """(db [N, V, d] on device, queries [Q, V, d] f32 on device, centroids)."""
    if w.storage == "float16":  # config 4: Zipf-skewed cells, fp16 storage
        db, qs, Ct = synth.zipf_mixture(w, SEED, device)
        return db, qs, Ct.cpu().numpy()
    db, qs, _labels = synth.mixture(w, SEED, device)
    return db, qs, synth.sample_centroids(db, w.K, SEED + 1).cpu().numpy()


def build(w, device):
    from paper_1604_01879_b200 import IndexConfig, build_index_from_views
    from paper_1604_01879_b200.codebook import Codebook

    if w.name == "c3":
        return build_streamed(w, device)
    db, qs, C = generate(w, device)
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


def host_oracle(bundle, w, single_channel=True):
    """oracle.OracleIndex over the (parity-verified) GPU-built lists: the CPU
    baseline inside the GPU arm (the reference arm builds its own index)."""
    import oracle

    fif = bundle.fifs["A"]
    ords, feats = fif.entry_ordinals, fif.entry_features
    raw = [oracle.Act(a.indices, a.values, a.norm) for a in bundle.raw_activations["A"]]
    sif = oracle.Sif(norms=bundle.sif.norms, entry_ordinals=bundle.sif.entry_ordinals,
                     entry_values=bundle.sif.entry_values)
    orc = oracle.OracleIndex.from_parts(
        bundle.shape_ids, fif.codebook.centroids, ords, feats, raw, sif, ma=w.ma, k1=w.k1,
        k2=w.k2, alpha=0.5, similarity="gaussian_expanded", sigma=w.sigma,
        single_channel=single_channel)
    for e in range(len(ords)):  # |p|^2 per cell, computed once before forking
        orc.fifs["A"].pnorm2(e)
    return orc


# forked CPU workers (oracle port of the reference path, one BLAS thread each)
_ORACLE = None
_QUERIES = None
_TOPK = 10


def _cpu_query(i):
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        res, _ = _ORACLE.query(_QUERIES[i], top_k=_TOPK, rerank=True)
    return len(res)


def cpu_sample(orc, queries_host, n_procs, n_queries, top_k):
    """Wall time of n_queries oracle queries on n_procs forked workers (or
    in this process, one BLAS thread, for n_procs = 1)."""
    import multiprocessing as mp

    global _ORACLE, _QUERIES, _TOPK
    _ORACLE, _QUERIES, _TOPK = orc, queries_host, top_k
    if n_procs == 1:
        _cpu_query(0)  # warm
        t0 = time.perf_counter()
        for i in range(n_queries):
            _cpu_query(i % len(queries_host))
        return time.perf_counter() - t0
    ctx = mp.get_context("fork")
    with ctx.Pool(n_procs) as pool:
        pool.map(_cpu_query, [0] * min(n_procs, 2))  # warm the forked workers
        t0 = time.perf_counter()
        pool.map(_cpu_query, [i % len(queries_host) for i in range(n_queries)], chunksize=1)
        return time.perf_counter() - t0


def _gpu_line(args, config, value, ms, scaling, e2e, launches, roofline, cpu, clk, run,
              dtype="f32"):
    ws, _, _ = dist_env()
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": config, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clk, "run": run}


def run_gift(args, w):
    """One index per rank: configs 1-2 at any N (replicas: disjoint query
    streams, no collective), other configs at N = 1."""
    from paper_1604_01879_b200 import query_many
    from paper_1604_01879_b200.index import GraphedQuery, lane_streams

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # init lines let the driver count the ranks
        dist.init_process_group("nccl", device_id=device)
    bundle, qs, build_s = build(w, device)
    eng = bundle.engine
    if args.drain_kb or args.pair != "auto":
        eng.fa.set_variant(drain_kb=args.drain_kb, pair=args.pair)
    _set_sif_mode(eng.sif, args)
    B = w.batch
    nb = max(1, qs.shape[0] // B)
    order = [(rank + i * ws) % nb for i in range(args.steps + args.warmup)]
    batches = [qs[j * B:(j + 1) * B].contiguous() for j in range(nb)]
    stream = torch.cuda.current_stream()
    # batch i runs on lane i % L: its own stream and scratch, so one batch's
    # quantize / reduce / re-rank kernels overlap the other batch's scan
    lanes_default, reserve_default = default_lanes(w.name)
    L = max(1, args.lanes if args.lanes is not None else lanes_default)
    # CUDA graphs: one replay per batch instead of ~34 launches from Python
    # (config 1's L2-resident batches issue faster than Python launches them)
    use_graph = args.graph == "on" or (args.graph == "auto" and w.name in GRAPH_CONFIGS)
    # (graph capture needs a side stream, also with one lane)
    lanes = [stream] if L == 1 and not use_graph else lane_streams(L)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    scan_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    for i, (a, b) in enumerate(scan_ev):  # torch creates CUDA events lazily, on first record
        a.record(lanes[i % L])
        b.record(lanes[i % L])
    # SMs the scan leaves to the other lanes' kernels
    eng.reserve_sms = (args.reserve_sms if args.reserve_sms is not None
                       else (reserve_default if L > 1 else 0))

    graphs = ([GraphedQuery(eng, batches[0], w.top_k, stream=s) for s in lanes]
              if use_graph else None)

    def step(i, bi, sev=None):
        s = lanes[i % L]
        if graphs is not None:
            graphs[i % L](batches[bi])
            return
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
    ms = ev[0].elapsed_time(ev[1])
    syncs = {}
    launches_per_step = count_launches(
        lambda: eng.run(batches[order[args.warmup]], top_k=w.top_k, rerank=True), syncs)
    # with batches in flight a scan's events also span its wait behind another
    # lane's scan: the kernel's own duration comes from the same batches run
    # one at a time right after, with the timed run's configuration (the same
    # SMs left to other lanes), inside the clock sampler's run
    scan_in_flight = [a.elapsed_time(b) for a, b in scan_ev] if graphs is None else None
    if L > 1 or graphs is not None:
        serial_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in range(args.steps)]
        for a, b in serial_ev:
            a.record(stream)
            b.record(stream)
        torch.cuda.synchronize()
        for i in range(args.steps):
            eng.run(batches[order[args.warmup + i]], top_k=w.top_k, rerank=True,
                    scan_events=serial_ev[i])
        torch.cuda.synchronize()
        scan_ms = [a.elapsed_time(b) for a, b in serial_ev]
    else:
        scan_ms = scan_in_flight
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_q = B * args.steps * ws
    value = total_q / (ms_max / 1000.0)

    # ---- e2e through the public API from pinned host memory: the timed
    # steps' batches, or the config's whole query set when that is larger
    # (config 2: "1,000 queries in batches of 64"; the pipeline's one batch of
    # fill latency is then spread over the workload the config names)
    if qs.shape[0] > args.steps * B:
        host = torch.empty(tuple(qs.shape), dtype=torch.float32, pin_memory=True)
        host.copy_(qs)
    else:
        host = torch.empty((args.steps * B, w.n_views, w.dim), dtype=torch.float32,
                           pin_memory=True)
        for i in range(args.steps):
            host[i * B:(i + 1) * B].copy_(batches[order[args.warmup + i]])
    e2e_q = host.shape[0]
    query_many(bundle, host[:L * B], top_k=w.top_k, lanes=L, reserve_sms=eng.reserve_sms,
               graph=use_graph)  # warm
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    query_many(bundle, host, top_k=w.top_k, lanes=L, reserve_sms=eng.reserve_sms,
               graph=use_graph)
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = e2e_q * ws / float(t.item())

    # ---- roofline of the dominant kernel (F-IF scan), per launch
    work = [scan_work(eng.fa, batches[order[args.warmup + i]], w, w.top_k)
            for i in range(args.steps)]
    nbytes = sum(x[0] for x in work) / len(work)
    flops = sum(x[1] for x in work) / len(work)
    scan_avg = sum(scan_ms) / len(scan_ms)
    roof = roofline_of(nbytes, flops, scan_avg, w, scan_kernel_name(w),
                       ("CUDA events around each scan launch, the timed batches re-run one "
                        f"at a time with the timed configuration ({eng.reserve_sms} SMs left "
                        "to other lanes)") if L > 1 else
                       "CUDA events around each scan launch inside the timed region",
                       q16=fp16_exact(batches[:4]))
    roof["scan_ms_in_flight_avg"] = (sum(scan_in_flight) / len(scan_in_flight)
                                     if scan_in_flight else None)
    roof["scan_share_of_step"] = scan_avg * args.steps / ms
    # lower bound independent of overlap: the scan's algorithmic bytes per
    # timed step (every step runs one scan) over the whole step time
    roof["achieved_gbs_per_step_lower_bound"] = nbytes / (ms / args.steps / 1000.0) / 1e9
    ncu = load_ncu(w.name)
    quant_ncu = ({"kernel": ncu["quantize_kernel"], "tensor_hmma_active_pct":
                  ncu["quantize_tensor_hmma_active_pct"], "source": "ncu --set full"}
                 if "quantize_kernel" in ncu else None)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and eng.fa.feat is not None:
        orc = host_oracle(bundle, w)
        qh = batches[0].cpu().numpy()
        cores = host_cores()
        wall = cpu_sample(orc, qh, cores, cores, w.top_k)
        cpu = {"value": cores / wall, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{cores} config-{w.name} queries on {cores} forked workers, one BLAS "
                         f"thread each (oracle port of query_fif + rerank_scores + ranking, "
                         f"single channel, over the GPU-built lists)", "host": host_info()}
    if rank == 0:
        run = {"lanes": L, "scan_reserved_sms": eng.reserve_sms, "build_s": build_s,
               "cuda_graph": bool(use_graph),
               "drain_kb": args.drain_kb or "default", "pair": args.pair,
               "host_blocking_cuda_calls_per_step": syncs,
               "features": ("planes only (streamed build)" if eng.fa.feat is None
                            else "storage copy + planes"), "quantize": quant_ncu}
        line = _gpu_line(args, workload_config(w, f"replicas{ws}" if ws > 1 else "single"),
                         value, ms_max / args.steps, "weak",
                         {"value": e2e_value, "unit": UNIT,
                          "h2d_bytes_per_step": B * w.n_views * w.dim * 4,
                          "d2h_bytes_per_step": B * w.top_k * 12,
                          "queries": e2e_q, "steps": -(-e2e_q // B)},
                         launches_per_step * args.steps, roof, cpu, clk.summary(), run)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init_dist(device):
    ws, _, _ = dist_env()
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # init lines let the driver count the ranks
        dist.init_process_group("nccl", device_id=device)
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)


def _timed_sharded(args, device, run_batch, n_batches, local):
    """Warm-up, then K steps bracketed by barrier + synchronize, device
    events; returns (max-over-ranks ms, clocks)."""
    ws, _, _ = dist_env()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with ClockSampler(local) as clk:
        warm(lambda i: run_batch(i % n_batches), args.warmup)
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        for i in range(args.steps):
            run_batch((args.warmup + i) % n_batches)
        ev[1].record()
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([ev[0].elapsed_time(ev[1])], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), clk.summary()


def _timed_sharded_many(args, device, eng, batches, top_k, lanes, local):
    """Like _timed_sharded, the K steps issued as batches in flight."""
    ws, _, _ = dist_env()
    nb = len(batches)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with ClockSampler(local) as clk:
        warm(lambda i: eng.run_many([batches[(i + j) % nb] for j in range(lanes)], top_k,
                                    lanes=lanes), args.warmup)  # every lane's scratch
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        eng.run_many([batches[(args.warmup + i) % nb] for i in range(args.steps)], top_k,
                     lanes=lanes)
        ev[1].record()
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([ev[0].elapsed_time(ev[1])], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), clk.summary()


def _e2e_sharded(device, host_batches, run_dev):
    """End to end through the sharded engine: every step copies its pinned
    host batch in, runs, and copies the merged top-k out (all inside)."""
    ws, _, _ = dist_env()
    bufs = [torch.empty_like(host_batches[0], device=device) for _ in range(2)]
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outs = None
    for i, hb in enumerate(host_batches):
        buf = bufs[i % 2]
        buf.copy_(hb, non_blocking=True)
        idx, val = run_dev(buf)
        if outs is None:  # pinned result buffers (a pageable D2H would block)
            outs = [(torch.empty(idx.shape, dtype=idx.dtype, pin_memory=True),
                     torch.empty(val.shape, dtype=val.dtype, pin_memory=True))
                    for _ in host_batches]
        outs[i][0].copy_(idx, non_blocking=True)
        outs[i][1].copy_(val, non_blocking=True)
    torch.cuda.synchronize()
    dist.barrier()
    e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    return float(e2e.item())


def run_sharded(args, w):
    """Database sharded by shape over the ranks (dist.py): every rank holds
    N / G shapes (all cells), queries are replicated, per-shard top-k2 and
    top-k candidates are merged with one packed NCCL all_gather each.  Every
    rank generates the seeded database itself (no broadcast of the
    self-join's query blocks)."""
    from paper_1604_01879_b200 import IndexConfig
    from paper_1604_01879_b200 import engine as eg
    from paper_1604_01879_b200.dist import ShardedEngine, build_sharded, shard_bounds

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    _init_dist(device)
    cfg = IndexConfig(n_views=w.n_views, codebook_size=w.K, ma=w.ma, k1=w.k1, k2=w.k2,
                      similarity="gaussian", sigma=w.sigma, storage_dtype=w.storage,
                      batch_size=w.batch, imported=True)
    lo, hi = shard_bounds(w.n_shapes, ws, rank)
    t0 = time.perf_counter()
    db = None
    if w.name.startswith("c3"):
        mix = synth.BlockMixture(w, SEED, device)
        C = synth.sample_centroids_rows(mix, w.K, SEED + 1).cpu().numpy()
        qs = mix.queries()
        X = mix.rows(lo, hi).to(cfg.torch_storage)
        query_views = mix.rows
    else:
        db, qs, C = generate(w, device)
        X = db[lo:hi].contiguous()
        query_views = lambda s0, s1: db[s0:s1]  # noqa: E731
    fif, raw, sif = build_sharded(X, eg.DeviceCodebook.from_numpy(C), cfg, w.n_shapes,
                                  batch=w.batch, query_views=query_views)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    del X, query_views, db
    torch.cuda.empty_cache()
    idrank = torch.arange(w.n_shapes, dtype=torch.int32, device=device)  # zero-padded ids
    eng = ShardedEngine(fif, raw, sif, idrank, cfg, w.n_shapes)
    B = w.batch
    nb = max(1, qs.shape[0] // B)
    batches = [qs[j * B:(j + 1) * B].contiguous() for j in range(nb)]
    # two batches in flight: batch i+1's quantize and scan overlap batch i's
    # exchanges (ShardedEngine.run_many); every rank issues the same order
    lanes = max(1, args.lanes or 2)
    ms, clk = _timed_sharded_many(args, device, eng, batches, w.top_k, lanes, local)
    syncs = {}
    launches = count_launches(lambda: eng.run(batches[0], w.top_k), syncs)
    steps = [batches[(args.warmup + i) % nb].cpu().pin_memory() for i in range(args.steps)]
    e2e_s = _e2e_sharded(device, steps, lambda q: eng.run(q, w.top_k))
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    for e in ev:  # torch creates CUDA events lazily, on first record
        e.record()
    sms = []
    for i in range(min(args.steps, 4)):
        eng.runner.score(fif, batches[i % nb], w.ma, eng.mode, w.sigma, cand_k=min(w.k2, 8),
                         dense=False, scan_events=ev)
        torch.cuda.synchronize()
        sms.append(ev[0].elapsed_time(ev[1]))
    work = [scan_work(fif, batches[i % nb], w, w.top_k) for i in range(min(args.steps, 4))]
    roof = roofline_of(sum(x[0] for x in work) / len(work), sum(x[1] for x in work) / len(work),
                       sum(sms) / len(sms), w, scan_kernel_name(w, " (this rank's shard)"),
                       "CUDA events around the shard's scan, batches run one at a time",
                       q16=fp16_exact(batches[:4]))
    if rank == 0:
        total_q = B * args.steps
        line = _gpu_line(args, workload_config(w, f"shard{ws}"), total_q / (ms / 1000.0),
                         ms / args.steps, "strong",
                         {"value": total_q / e2e_s, "unit": UNIT,
                          "h2d_bytes_per_step": B * w.n_views * w.dim * 4,
                          "d2h_bytes_per_step": B * w.top_k * 12},
                         launches * args.steps, roof, None, clk,
                         {"build_s": build_s, "shard_shapes": hi - lo, "lanes": lanes,
                          "host_blocking_cuda_calls_per_step": syncs,
                          "collectives_per_step": 2 if ws > 1 else 0,
                          "exchange": "packed all_gather_into_tensor (score bits, "
                                      "ordinal << 32 | tiebreak) + gift_topk_cand_tb merge"})
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _set_sif_mode(sif, args):
    """--sif: force one S-IF query implementation (default: by batch size)."""
    from paper_1604_01879_b200 import _native as nat

    sif.query_flags = {"auto": 0, "rows": nat.SIF_ROWS, "sort": nat.SIF_SORT,
                       "bucket": nat.SIF_BUCKET}[args.sif]


C5_LANES = 3  # config 5: S-IF query batches in flight (latency-bound kernels; 1..4: 401k, 468k, 488k, 478k q/s)


def run_c5(args):
    """Config 5 (re-rank dominated): given top-50 lists for 1M shapes, S-IF
    over all shapes, queries re-ranked with k = 50 neighbour-set Jaccard.
    N > 1 (or --shard): the S-IF sharded by shape, one packed all-gather of
    the per-shard top-100 per batch."""
    from paper_1604_01879_b200 import IndexConfig, build_index_from_lists

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    c = synth.C5
    n = args.c5_shapes or c["n_shapes"]
    idx, val = synth.community_lists(SEED, device, n_shapes=n, communities=c5_communities(n))
    cfg = IndexConfig(k1=c["list_len"], k2=c["k2"], imported=True, batch_size=c["batch"])
    g = torch.Generator(device=device)
    g.manual_seed(SEED + 5)
    B = c["batch"]
    nsteps = args.steps + args.warmup
    qrows = torch.randint(0, n, (B * nsteps,), generator=g, device=device)
    sharded = ws > 1 or args.shard
    bundle = None
    t0 = time.perf_counter()
    if sharded:
        from paper_1604_01879_b200.dist import ShardedEngine, build_sharded_from_lists

        _init_dist(device)
        raw, sif = build_sharded_from_lists(idx, val, cfg)
        _set_sif_mode(sif, args)
        eng = ShardedEngine(None, raw, sif, torch.arange(n, dtype=torch.int32, device=device),
                            cfg, n)

        def run_q(qi, qv, r):
            return eng.rerank_lists(qi, qv, c["top_k"], self_global=r)
        postings = int(sif.e_ord.numel())
    else:
        bundle = build_index_from_lists(idx, val, synth.shape_ids(n), cfg)
        eng = bundle.engine
        _set_sif_mode(eng.sif, args)

        def run_q(qi, qv, r):
            return eng.rerank_lists(qi, qv, top_k=c["top_k"], self_local=r.to(torch.int32))
        postings = int(bundle.sif.dev.e_ord.numel())
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    rows = [qrows[i * B:(i + 1) * B] for i in range(nsteps)]
    step = lambda j: run_q(idx[rows[j]], val[rows[j]], rows[j])  # noqa: E731
    if sharded:
        ms, clk = _timed_sharded(args, device, step, nsteps, local)
    else:
        # batches in flight: batch i on lane stream i % L (each lane keeps its
        # own S-IF workspace and accumulator rows), as query_many does
        from paper_1604_01879_b200.index import lane_streams

        n_lanes = max(1, args.lanes if args.lanes is not None else C5_LANES)
        lanes = lane_streams(n_lanes)
        main = torch.cuda.current_stream()

        def run_lanes(indices):
            for s in lanes:
                s.wait_stream(main)
            for n_, i in enumerate(indices):
                with torch.cuda.stream(lanes[n_ % n_lanes]):
                    step(i)
            for s in lanes:
                main.wait_stream(s)

        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with ClockSampler(local) as clk_s:
            warm(lambda i: run_lanes([i % args.warmup] * n_lanes), args.warmup)
            ev[0].record()
            run_lanes(range(args.warmup, nsteps))
            ev[1].record()
            torch.cuda.synchronize()
        ms, clk = ev[0].elapsed_time(ev[1]), clk_s.summary()
    syncs = {}
    launches = count_launches(lambda: step(0), syncs)
    # e2e: each step's given lists come from pinned host memory, results go back
    host = [(idx[r].cpu().pin_memory(), val[r].cpu().pin_memory(), r.cpu().pin_memory())
            for r in rows[args.warmup:]]
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    k_out = c["top_k"]
    res = [(torch.empty((B, k_out), dtype=torch.int32, pin_memory=True),
            torch.empty((B, k_out), dtype=torch.float64, pin_memory=True)) for _ in host]
    e_lanes = lanes if not sharded else [torch.cuda.current_stream()]
    t0 = time.perf_counter()
    for n_, ((hi_, hv, hr), (ri, rv)) in enumerate(zip(host, res)):
        with torch.cuda.stream(e_lanes[n_ % len(e_lanes)]):  # copies and compute per lane
            oi, ov = run_q(hi_.to(device, non_blocking=True), hv.to(device, non_blocking=True),
                           hr.to(device, non_blocking=True))
            ri.copy_(oi, non_blocking=True)
            rv.copy_(ov, non_blocking=True)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if sharded:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    roof = None
    if bundle is not None:
        roof = c5_roofline(bundle, idx, val, rows[args.warmup:args.warmup + min(args.steps, 4)], c)
    cpu = None
    if rank == 0 and bundle is not None and not args.no_cpu_baseline:
        cpu = c5_cpu_baseline(bundle, idx, val, rows[args.warmup], c)
    if rank == 0:
        L = c["list_len"]
        line = _gpu_line(args, c5_config(c, n, f"shard{ws}" if sharded else "single"),
                         B * args.steps / (ms / 1000.0), ms / args.steps,
                         "strong" if sharded else "weak",
                         {"value": B * args.steps / e2e_s, "unit": UNIT,
                          "h2d_bytes_per_step": B * (L * 12 + 8),
                          "d2h_bytes_per_step": B * c["top_k"] * 12},
                         launches * args.steps, roof, cpu, clk,
                         {"build_s": build_s, "sif_postings": postings,
                          "lanes": 1 if sharded else n_lanes,
                          "host_blocking_cuda_calls_per_step": syncs}, dtype="f64")
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


def c5_roofline(bundle, idx, val, rows, c):
    """Roofline of config 5's dominant step, the S-IF query + ranking of a
    batch (gift_sif_query_topk: bucket split of the touched postings by shape
    range, shared-memory sums, top-100): algorithmic bytes = the postings of
    the query activations' coordinates, 12 B each (i32 owner + f64 value:
    one read of every touched posting, rerank.py:187-230); time = CUDA events
    around the call, the timed batches re-run one at a time."""
    from paper_1604_01879_b200 import engine as eg

    eng = bundle.engine
    e_off = bundle.sif.dev.e_off
    lens = e_off[1:] - e_off[:-1]
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    nbytes, ms = [], []
    for r in rows:
        qi, qv = idx[r], val[r]
        k2 = min(eng.cfg.k2, qi.shape[1])
        nbr = torch.where(qv[:, :k2] > 0, qi[:, :k2], torch.full_like(qi[:, :k2], -1))
        fa = eg.act_mean(eng.raw_a, nbr.to(torch.int32).contiguous())
        live = torch.arange(fa.cap, device=fa.idx.device)[None, :] < fa.cnt[:, None].long()
        nbytes.append(float(lens[fa.idx[live].long()].sum().item()) * 12.0)
        torch.cuda.synchronize()
        ev[0].record()
        eng._sif_rank(fa, c["top_k"], r.to(torch.int32))
        ev[1].record()
        torch.cuda.synchronize()
        ms.append(ev[0].elapsed_time(ev[1]))
    peak, peak_kind = measured_peaks()
    b = sum(nbytes) / len(nbytes)
    t = sum(ms) / len(ms)
    achieved = b / (t / 1000.0) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "kernel": "gift_sif_query_topk (sif_split_* + bucket sums + "
            "ranking kernels)", "peak_source": peak_kind, "traffic": None,
            "alg_bytes_per_launch": b, "sif_ms_avg": t,
            "measured": "CUDA events around the S-IF query + ranking of each timed batch, "
                        "re-run one at a time"}


_C5 = None


def _c5_query(i):
    import oracle

    raw, sif, ids, qi, qv, r, n, c = _C5
    scores = np.zeros(n)
    scores[qi[i]] = qv[i]
    nb = oracle.top_neighbors(scores, c["k2"])
    f = oracle.mean_activation(raw, nb)
    fin = oracle.query_sif(sif, oracle.aggregate(f, f, 0.5))
    return oracle.lexsort_rank(fin, ids, ids[r[i]], c["top_k"])[:1].tolist()


def c5_cpu_baseline(bundle, idx, val, rows, c):
    """The reference's query-time path for config 5 (index.py:249-299 from
    given lists: top_neighbors over the dense score row, mean_activation,
    aggregate, query_sif, lexsort ranking over all shapes) on the host cores,
    over the GPU-built raw activations and S-IF (oracle port, forked
    workers)."""
    import multiprocessing as mp

    import oracle

    global _C5
    raw = [oracle.Act(a.indices, a.values, a.norm) for a in bundle.raw_activations["A"]]
    sif = oracle.Sif(norms=bundle.sif.norms, entry_ordinals=bundle.sif.entry_ordinals,
                     entry_values=bundle.sif.entry_values)
    ids = np.asarray(bundle.shape_ids)
    r = rows.cpu().numpy()
    _C5 = (raw, sif, ids, idx[rows].cpu().numpy(), val[rows].cpu().numpy(), r, len(raw), c)
    cores = host_cores()
    nq = 2 * cores
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_c5_query, [0] * cores)
        t0 = time.perf_counter()
        pool.map(_c5_query, [i % len(r) for i in range(nq)], chunksize=1)
        wall = time.perf_counter() - t0
    return {"value": nq / wall, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{nq} config-5 queries on {cores} forked workers (oracle port of "
                      f"rerank_scores + ranking over dense rows of all shapes, GPU-built S-IF)",
            "host": host_info()}


# ------------------------------------------------------------------ reference arm
def reference_index(w, device):
    """The index of configs 1-2 built on the HOST by the oracle: the seeded
    workload (the GPU arm's own generator; torch only), every view quantized
    bit-exactly, the lists laid out, the full f64 self-join, co-augment and
    the S-IF (oracle/scale.py).  No product code runs."""
    import oracle
    from oracle import scale

    db, qs, C = generate(w, device)
    db_h = db.cpu().numpy()
    qs_h = qs.cpu().numpy()
    del db, qs
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    idx = scale.OracleCsrIndex.from_views(db_h, C, w.ma, w.k1, w.k2, "gaussian", w.sigma)
    build_s = time.perf_counter() - t0
    off = idx.cell_off
    ords = [idx.post_ord[off[c]:off[c + 1]] for c in range(w.K)]
    feats = [idx.feat[off[c]:off[c + 1]] for c in range(w.K)]
    ids = synth.shape_ids(w.n_shapes)
    per = {}
    for single in (True, False):
        per[single] = oracle.OracleIndex.from_parts(
            ids, C, ords, feats, idx.raw, idx.sif, ma=w.ma, k1=w.k1, k2=w.k2,
            similarity="gaussian_expanded", sigma=w.sigma, single_channel=single)
    for e in range(w.K):  # |p|^2 per cell, once, before forking (shared Fif)
        per[True].fifs["A"].pnorm2(e)
    return per, qs_h, build_s


def run_reference(args, w):
    ws, rank, local = dist_env()
    if ws > 1 and rank != 0:
        return
    if w.name not in ("c1", "c2"):
        print(json.dumps({"impl": "reference", "unavailable":
                          f"config {w.name}: the host build of the reference index (bit-exact "
                          "quantize of every view + the f64 self-join) takes hours; its CPU "
                          "baseline is the GPU arm's cpu_baseline over GPU-built lists"}))
        return
    torch.cuda.set_device(local)
    per, qh, build_s = reference_index(w, torch.device("cuda", local))
    cores = host_cores()
    orc = per[True]
    for _ in range(min(args.warmup, 1)):  # forks + page-ins; one step suffices on the CPU
        cpu_sample(orc, qh, cores, cores, w.top_k)
    times = [cpu_sample(orc, qh, cores, cores, w.top_k) for _ in range(args.steps)]
    qps = cores * len(times) / sum(times)
    as_is_s = cpu_sample(per[False], qh, cores, cores, w.top_k)
    lat_q = 2
    lat_s = cpu_sample(orc, qh, 1, lat_q, w.top_k)
    sample = (f"{cores} queries/step x {len(times)} steps of config {w.name} on {cores} forked "
              f"workers, one BLAS thread each: the oracle port of the reference's query "
              f"(quantize, query_fif with one f64 GEMV per probed cell, rerank_scores, lexsort "
              f"ranking), single channel; over an index the oracle built on the host in "
              f"{build_s:.0f} s")
    line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(w, f"replicas{ws}" if ws > 1 else "single"),
            "cpu_baseline": {"value": qps, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample, "host": host_info(),
                             "as_is_two_channel_qps": cores / as_is_s,
                             "latency_1core_ms": 1000 * lat_s / lat_q,
                             "index_build_s": build_s},
            "e2e": {"value": qps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main
def _relaunch(n):
    """--gpus N without torchrun: one rank per GPU via torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


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
                    help="SMs the scan leaves to other lanes (default per config)")
    ap.add_argument("--lanes", type=int, default=None,
                    help="batches in flight on separate streams (1 = serial; default per config)")
    ap.add_argument("--drain-kb", type=int, default=0,
                    help="scan accumulator drain interval in 64-wide k-blocks (0 = the "
                         "library default)")
    ap.add_argument("--pair", default="auto", choices=["auto", "on", "off"],
                    help="F-IF scan on CTA pairs (cta_group::2): default per storage")
    ap.add_argument("--sif", default="auto", choices=["auto", "rows", "sort", "bucket"],
                    help="S-IF query implementation (default: by batch size)")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay each lane's query pipeline as a CUDA graph (default: config 1)")
    ap.add_argument("--shard", action="store_true",
                    help="shard the database by shape over the ranks (default for configs "
                         "3-5 at N > 1)")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and args.gpus > 1:
        _relaunch(args.gpus)
    if ws and ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    args.warmup = max(args.warmup, 3) if args.impl == "gift" else args.warmup
    if args.config == "c5":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable":
                              "config 5: the host build of the reference S-IF over 1M shapes "
                              "(dict loops) takes tens of minutes; its CPU baseline is the GPU "
                              "arm's cpu_baseline over the GPU-built S-IF"}))
            return
        run_c5(args)
        return
    w = synth.WORKLOADS[args.config]
    if args.impl == "reference":
        run_reference(args, w)
    elif args.shard or (args.gpus > 1 and w.name not in ("c1", "c2")):
        run_sharded(args, w)
    else:
        run_gift(args, w)


if __name__ == "__main__":
    main()
