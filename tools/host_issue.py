"""Host-side issue cost of one query batch (C2) vs its device time."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
w = bench.synth.WORKLOADS["c2"]
dev = torch.device("cuda", 0)
bundle, qs, _ = bench.build(w, dev)
eng = bundle.engine
B = w.batch
batches = [qs[j * B:(j + 1) * B].contiguous() for j in range(8)]
for i in range(10):
    eng.run(batches[i % 8], top_k=w.top_k)
torch.cuda.synchronize()
# host issue time with the GPU busy (queue never drains)
big = torch.empty(1 << 28, device=dev)
for rep in range(3):
    big.fill_(1.0)  # keep the device busy ~ a few ms
    t0 = time.perf_counter()
    for i in range(20):
        eng.run(batches[i % 8], top_k=w.top_k)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host issue {1000 * (t1 - t0) / 20:.3f} ms/batch, wall {1000 * (t2 - t0) / 20:.3f} ms/batch")
