"""How many views of a bench query batch need the exact quantize re-check
(candidates under (ma-th smallest approx) + 2M), and the time of the
quantize call alone:  python tools/quant_flags.py c2"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1604_01879_b200 import engine as eg  # noqa: E402
from paper_1604_01879_b200 import synth  # noqa: E402

w = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dev = torch.device("cuda", 0)
bundle, qs, _ = bench.build(w, dev)
cb = bundle.engine.fa.cb
X = qs[: w.batch].reshape(-1, w.dim).double()
C = cb.centroids.double()
ap = (C * C).sum(1)[None] - 2 * X @ C.T
s, _ = ap.sort(1)
M = 1.5 * 2 * 1.45e-5
kth = s[:, w.ma - 1]
cnt = (ap <= (kth + 2 * M)[:, None]).sum(1)
print("views", X.shape[0], "flagged", int((cnt > w.ma).sum()), "max cnt", int(cnt.max()),
      "hist", torch.bincount(cnt.cpu())[:12].tolist())
flat = qs[: w.batch].reshape(-1, w.dim).contiguous()
for _ in range(3):
    eg.quantize_rows(cb, flat, w.ma)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    eg.quantize_rows(cb, flat, w.ma)
e1.record()
torch.cuda.synchronize()
print("quantize ms", e0.elapsed_time(e1) / 10)
