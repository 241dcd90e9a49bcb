"""Feature-ingest throughput: a synthetic GIFTFT1 file
(config-2 rows, d = 4096) written to /tmp, then
  * device: FeatureFile.device_rows of every shape (host gather + f64 norms,
    H2D, GPU normalization), GB/s of file payload, synchronized;
  * host: the package's import_features restatement (the reference's
    algorithm, per-row Python objects) on a sample of shapes.
    python tools/ingest_bench.py [--shapes 2000]"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_01879_b200 import features as ft  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", type=int, default=2000)
ap.add_argument("--views", type=int, default=64)
ap.add_argument("--dim", type=int, default=4096)
ap.add_argument("--sample", type=int, default=64)
args = ap.parse_args()
rng = np.random.default_rng(5)
with tempfile.TemporaryDirectory() as td:
    p = os.path.join(td, "feat.bin")
    with open(p, "wb") as fh:
        import struct
        fh.write(ft.FEATURE_MAGIC + struct.pack("<I", args.shapes))
        blk = np.abs(rng.standard_normal((args.views, args.dim))).astype("<f4")
        for i in range(args.shapes):
            sid = f"s{i:07d}".encode()
            fh.write(struct.pack("<H", len(sid)) + sid + struct.pack("<II", args.views, args.dim))
            blk[i % args.views] += np.float32(0.5)
            fh.write(blk.tobytes())
    payload = args.shapes * args.views * args.dim * 4
    f = ft.FeatureFile(p, "A")
    torch.cuda.set_device(0)
    f.device_rows(range(min(64, len(f))))  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = f.device_rows(range(len(f)))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ns = min(args.sample, args.shapes)
    sub = os.path.join(td, "sample.bin")
    with open(sub, "wb") as fh:
        fh.write(ft.FEATURE_MAGIC + struct.pack("<I", ns))
        with open(p, "rb") as src:
            src.seek(12)
            for _ in range(ns):
                (n,) = struct.unpack("<H", src.read(2))
                fh.write(struct.pack("<H", n) + src.read(n))
                hdr = src.read(8)
                nv, d = struct.unpack("<II", hdr)
                fh.write(hdr + src.read(nv * d * 4))
    t1 = time.perf_counter()
    ft.import_features(sub, "A")
    dh = time.perf_counter() - t1
    print(json.dumps({"metric": "feature ingest GB/s (GIFTFT1 payload)", "shapes": args.shapes,
                      "payload_gb": payload / 1e9, "device_gbs": payload / dt / 1e9,
                      "device_s": dt, "host_import_gbs": ns * args.views * args.dim * 4 / dh / 1e9,
                      "host_sample_shapes": ns, "cores": 1}))
