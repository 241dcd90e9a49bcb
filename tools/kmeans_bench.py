"""Codebook training throughput: device
train_codebook vs the reference algorithm on the host (the oracle port, the
reference's own numpy/BLAS calls), same seeded mixture rows.
    python tools/kmeans_bench.py [--n 20000 --d 256 --k 64 --iters 10]"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from cases import mixture_views  # noqa: E402
from paper_1604_01879_b200.codebook import train_codebook  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=20000)
ap.add_argument("--d", type=int, default=256)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
x, _ = mixture_views(9, args.n // 10, 10, args.d, 40, sigma=0.5)
x = x.reshape(-1, args.d).astype(np.float64)
torch.cuda.set_device(0)
train_codebook(x[:1000], 8, seed=1, max_iters=2)  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
cb = train_codebook(x, args.k, seed=3, max_iters=args.iters)
torch.cuda.synchronize()
dev_s = time.perf_counter() - t0
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: the reference algorithm on the host)

t0 = time.perf_counter()
ref = oracle.train_codebook(x, args.k, 3, args.iters)
host_s = time.perf_counter() - t0
print(json.dumps({"metric": "codebook training seconds (k-means++ + Lloyd, f64)",
                  "n": x.shape[0], "d": args.d, "k": args.k, "max_iters": args.iters,
                  "device_s": dev_s, "host_reference_s": host_s, "speedup": host_s / dev_s,
                  "identical_centroids": bool(np.array_equal(cb.centroids, ref)),
                  "host_threads": os.cpu_count()}))
