"""Timing experiments on the scan's pipeline roles (EXPERIMENT BUILD ONLY:
tools/libgift_exp.so, compiled with -DGIFT_SCAN_EXPERIMENT; outputs invalid).
Copies the experiment library over the in-tree libgift.so on the GPU box."""
import ctypes
import os
import shutil
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
shutil.copy(os.path.join(ROOT, "tools", "libgift_exp.so"),
            os.path.join(ROOT, "paper_1604_01879_b200", "libgift.so"))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1604_01879_b200 import _native as nat, engine as eg, matching as mt, synth  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402

lib = nat.lib()
lib.gift_scan_experiment.argtypes = [ctypes.c_int]
dev = torch.device("cuda", 0)
name = sys.argv[1] if len(sys.argv) > 1 else "c4s"
w = synth.WORKLOADS[name]
if w.storage == "float16":
    db, qs, Ct = synth.zipf_mixture(w, 20160407, dev)
    C = Ct.cpu().numpy()
else:
    db, qs, _ = synth.mixture(w, 20160407, dev)
    C = synth.sample_centroids(db, w.K, 20160408).cpu().numpy()
fif = mt.build_fif_from_tensor(db, Codebook(C), synth.shape_ids(w.n_shapes))
del db
q = qs[:w.batch].contiguous()
run = eg.ScoreRunner()
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
for e in ev:
    e.record()
run.score(fif.dev, q, w.ma, nat.SIM_GAUSSIAN, 0.5, cand_k=4, dense=False)
torch.cuda.synchronize()
meta = next(iter(run._ws.values())).get(64)[:64].view(torch.int64).cpu().tolist()
print(f"{name} items {meta[0]} compact {meta[1]} tiles {fif.dev.T} postings {fif.dev.P} "
      f"segments {fif.dev.S} queries {q.shape[0]}", flush=True)
for bits, label in ((0, "full"), (1, "no tail"), (2, "no drains"), (3, "no drains, no tail"),
                    (4, "no MMAs"), (5, "no MMAs, no tail"), (8, "no loads"),
                    (9, "no loads, no tail"), (11, "MMAs only"), (7, "loads only"),
                    (13, "drains only"), (14, "tail only"), (15, "nothing (scheduling only)")):
    lib.gift_scan_experiment(bits)
    ts = []
    for i in range(6):
        run.score(fif.dev, q, w.ma, nat.SIM_GAUSSIAN, 0.5, cand_k=4, dense=False, scan_events=ev)
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    print(f"{name} {label:28s} scan {sorted(ts)[len(ts) // 2]:.3f} ms", flush=True)
