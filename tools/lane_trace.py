"""Kernel timeline of the bench loop with batches in flight (CUPTI via
torch.profiler): how much of the wall time has a scan running, and which
kernels run while no scan does (the part the lanes do not hide).
    python tools/lane_trace.py --config c2 --lanes 4 --steps 12"""
import argparse
import collections
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1604_01879_b200 import synth  # noqa: E402
from paper_1604_01879_b200.index import lane_streams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--lanes", type=int, default=4)
ap.add_argument("--steps", type=int, default=12)
args = ap.parse_args()
w = synth.WORKLOADS[args.config]
torch.cuda.set_device(0)
bundle, qs, _ = bench.build(w, torch.device("cuda", 0))
eng = bundle.engine
B = w.batch
batches = [qs[j * B:(j + 1) * B].contiguous() for j in range(max(1, qs.shape[0] // B))]
L = args.lanes
lanes = [torch.cuda.current_stream()] if L == 1 else lane_streams(L)


def run(n):
    main = torch.cuda.current_stream()
    for s in lanes:
        s.wait_stream(main)
    for i in range(n):
        with torch.cuda.stream(lanes[i % L]):
            eng.run(batches[i % len(batches)], top_k=w.top_k, rerank=True)
    for s in lanes:
        main.wait_stream(s)
    torch.cuda.synchronize()


run(2 * L)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run(args.steps)
ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
t0 = min(a for a, _, _ in iv)
t1 = max(b for _, b, _ in iv)
pts = sorted({a for a, _, _ in iv} | {b for _, b, _ in iv})
scan_t = other_only = idle = 0.0
alone = collections.Counter()
for a, b in zip(pts, pts[1:]):
    act = [n for s, e, n in iv if s <= a and e >= b]
    d = b - a
    if any("fif_scan" in n for n in act):
        scan_t += d
    elif act:
        other_only += d
        for n in act:
            alone[n.split("(")[0][-40:]] += d / len(act)
    else:
        idle += d
per_kernel = collections.Counter()
for s_, e_, n in iv:
    per_kernel[n.split("(")[0][-48:]] += (e_ - s_) / args.steps
print(json.dumps({"config": w.name, "lanes": L, "steps": args.steps,
                  "kernel_us_per_step": [[k, round(v, 1)] for k, v in per_kernel.most_common(16)],
                  "wall_us_per_step": (t1 - t0) / args.steps,
                  "scan_active_us_per_step": scan_t / args.steps,
                  "no_scan_busy_us_per_step": other_only / args.steps,
                  "idle_us_per_step": idle / args.steps,
                  "busy_without_scan_top": [[k, round(v / args.steps, 1)]
                                            for k, v in alone.most_common(12)]}))
