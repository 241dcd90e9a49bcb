"""Per-stage device time of the single-channel query pipeline (CUDA events on
the launching stream, inputs resident), for one bench workload:

    python tools/stage_profile.py --config c4 [--steps 5]

Stages follow QueryEngine.run's fast path: quantize (timed alone, the same
call the score ABI makes first), score = view prep + quantize + plan + scan +
reduce (the scan bracketed by its own events), top-k2 candidate merge,
activation mean, S-IF query, final top-k.  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1604_01879_b200 import engine as eg  # noqa: E402
from paper_1604_01879_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--kernels", action="store_true",
                    help="also print per-kernel device time (torch.profiler / CUPTI)")
    ap.add_argument("--no-quantize", action="store_true",
                    help="skip the separately timed quantize call (kernel totals = pipeline only)")
    ap.add_argument("--reduce", default="gather,range",
                    help="comma list of reduce implementations to time (GIFT_REDUCE)")
    args = ap.parse_args()
    w = synth.WORKLOADS[args.config]
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    bundle, qs, build_s = bench.build(w, dev)
    eng = bundle.engine
    B = w.batch
    batches = [qs[j * B:(j + 1) * B].contiguous() for j in range(max(1, qs.shape[0] // B))]
    for impl in args.reduce.split(","):
        os.environ["GIFT_REDUCE"] = impl
        profile(eng, w, batches, args.steps, impl, build_s, not args.no_quantize)
        if args.kernels:
            from torch.profiler import ProfilerActivity
            from torch.profiler import profile as tprof

            with tprof(activities=[ProfilerActivity.CUDA]) as prof:
                profile(eng, w, batches, args.steps, impl + "+cupti", build_s,
                        not args.no_quantize)
            rows = []
            for e in prof.key_averages():
                t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
                if t > 0:
                    rows.append((t / (args.steps + 2) / 1000.0, e.count // (args.steps + 2),
                                 e.key[:90]))
            rows.sort(reverse=True)
            print(json.dumps({"config": w.name, "reduce": impl, "kernels_ms_per_step":
                              [[round(t, 4), c, k] for t, c, k in rows[:25]]}), flush=True)


def profile(eng, w, batches, steps, impl, build_s, quant=True):
    B = w.batch
    names = ["quantize", "score", "scan", "topk_cand", "act_mean", "sif_query", "topk_final"]
    tot = {n: 0.0 for n in names}
    k2 = min(eng.cfg.k2, eng.n)
    for it in range(steps + 2):
        Q = batches[it % len(batches)]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
        sev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for e in sev:  # torch creates CUDA events lazily, on first record
            e.record()
        flat = Q.reshape(-1, Q.shape[-1])
        ev[0].record()
        if quant:
            nz, _ = eg.view_prep(flat)
            eg.quantize_rows(eng.fa.cb, flat, eng.cfg.ma, nz=nz)
        ev[1].record()
        _, cs, ci = eng.runner.score(eng.fa, Q, eng.cfg.ma, eng.mode, eng.cfg.sigma,
                                     scan_events=sev, cand_k=k2, dense=False)
        ev[2].record()
        nbr, _ = eg.topk_candidates(cs, ci, k2, positive_only=True)
        ev[3].record()
        fa = eg.act_mean(eng.raw_a, nbr)
        ev[4].record()
        ev[5].record()
        eng._sif_rank(fa, w.top_k)  # sparse S-IF query + final ranking
        ev[6].record()
        torch.cuda.synchronize()
        if it < 2:
            continue
        tot["quantize"] += ev[0].elapsed_time(ev[1])
        tot["score"] += ev[1].elapsed_time(ev[2])
        tot["scan"] += sev[0].elapsed_time(sev[1])
        tot["topk_cand"] += ev[2].elapsed_time(ev[3])
        tot["act_mean"] += ev[3].elapsed_time(ev[4])
        tot["sif_query"] += ev[4].elapsed_time(ev[5])
        tot["topk_final"] += ev[5].elapsed_time(ev[6])
    ms = {k: v / steps for k, v in tot.items()}
    ms["score_minus_scan_minus_quantize"] = ms["score"] - ms["scan"] - ms["quantize"]
    print(json.dumps({"config": w.name, "reduce": impl, "batch": B, "build_s": build_s,
                      "ms": ms}), flush=True)


if __name__ == "__main__":
    main()
