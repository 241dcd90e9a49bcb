"""CUDA-graph replay of QueryEngine.run vs eager (config 1 / 2): identical
results, per-batch time."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1604_01879_b200 import synth  # noqa: E402
from paper_1604_01879_b200.index import GraphedQuery  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = synth.WORKLOADS[name]
dev = torch.device("cuda", 0)
bundle, qs, _ = bench.build(w, dev)
eng = bundle.engine
B = w.batch
batches = [qs[j * B:(j + 1) * B].contiguous() for j in range(qs.shape[0] // B)]
gq = GraphedQuery(eng, batches[0], w.top_k)
for b in batches[:6]:
    ei, ev = eng.run(b, top_k=w.top_k, rerank=True)
    gi, gv = gq(b)
    torch.cuda.synchronize()
    assert torch.equal(ei, gi) and torch.equal(ev, gv), "graph replay differs"
print("identical on 6 batches")
for label, fn in (("eager", lambda b: eng.run(b, top_k=w.top_k, rerank=True)), ("graph", gq)):
    for _ in range(3):
        fn(batches[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 50
    for i in range(n):
        fn(batches[i % len(batches)])
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{name} {label}: {dt * 1e3:.3f} ms per batch of {B} ({B / dt:.0f} q/s, one stream)")
