"""Per-kernel device time of config-5 re-rank batches (torch.profiler / CUPTI)."""
import json
import os
import sys

import torch

ROOT = os.getcwd()
sys.path.insert(0, ROOT)
from paper_1604_01879_b200 import IndexConfig, build_index_from_lists, synth  # noqa: E402

dev = torch.device("cuda", 0)
c = synth.C5
n = c["n_shapes"]
idx, val = synth.community_lists(20160407, dev, n_shapes=n)
bundle = build_index_from_lists(idx, val, synth.shape_ids(n),
                                IndexConfig(k1=c["list_len"], k2=c["k2"], imported=True,
                                            batch_size=c["batch"]))
eng = bundle.engine
B = c["batch"]
g = torch.Generator(device=dev)
g.manual_seed(5)
rows = torch.randint(0, n, (B * 8,), generator=g, device=dev)
for i in range(3):
    r = rows[i * B:(i + 1) * B]
    eng.rerank_lists(idx[r], val[r], top_k=100, self_local=r.to(torch.int32))
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(3, 6):
        r = rows[i * B:(i + 1) * B]
        eng.rerank_lists(idx[r], val[r], top_k=100, self_local=r.to(torch.int32))
    torch.cuda.synchronize()
out = []
for e in prof.key_averages():
    t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
    if t > 0:
        out.append([round(t / 3 / 1000.0, 4), e.count // 3, e.key[:70]])
out.sort(reverse=True)
print(json.dumps({"max_list": eng.sif.max_list, "kernels_ms_per_batch": out[:10]}))
