"""Per-role timeline of the tensor-core scan (EXPERIMENT BUILD ONLY:
tools/libgift_exp.so, -DGIFT_SCAN_EXPERIMENT).  The first 8 CTAs stamp
clock64 per item at: 0 scheduler published, 1 producer took, 2 producer
issued its last stage, 3 MMA took, 4 MMA committed its last chunk, 5 epilogue
took, 6 epilogue drained, 7 epilogue tail done (8 = N, 9 = cell).  Writes the
raw stamps to gpurun_out/trace_<config>.npy and prints per-role busy times."""
import ctypes
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
shutil.copy(os.path.join(ROOT, "tools", "libgift_exp.so"),
            os.path.join(ROOT, "paper_1604_01879_b200", "libgift.so"))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1604_01879_b200 import _native as nat, engine as eg, matching as mt, synth  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402

lib = nat.lib()
lib.gift_scan_trace.argtypes = [ctypes.c_void_p]
lib.gift_scan_experiment.argtypes = [ctypes.c_int]
dev = torch.device("cuda", 0)
name = sys.argv[1] if len(sys.argv) > 1 else "c4s"
drain = int(sys.argv[2]) if len(sys.argv) > 2 else 0
expbits = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kern = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # 0: posting-major scan, 1: dense cells
w = synth.WORKLOADS[name]
if w.storage == "float16":
    db, qs, Ct = synth.zipf_mixture(w, 20160407, dev)
    C = Ct.cpu().numpy()
else:
    db, qs, _ = synth.mixture(w, 20160407, dev)
    C = synth.sample_centroids(db, w.K, 20160408).cpu().numpy()
fif = mt.build_fif_from_tensor(db, Codebook(C), synth.shape_ids(w.n_shapes))
del db
fif.dev.set_variant(drain_kb=drain)
q = qs[:w.batch].contiguous()
so = fif.dev.seg_off.cpu().numpy()
co = fif.dev.cell_off.cpu().numpy()
big = np.argsort(-(co[1:] - co[:-1]))[:6]
print("largest cells (postings, segments):",
      [(int(co[c + 1] - co[c]), int(so[c + 1] - so[c])) for c in big], flush=True)
print(f"{name} postings {fif.dev.P} segments {fif.dev.S} tiles {fif.dev.T} "
      f"avg segment length {fif.dev.P / max(fif.dev.S, 1):.2f}", flush=True)
run = eg.ScoreRunner()
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
for e in ev:
    e.record()
TR = torch.zeros(2 * 8 * 512 * 16, dtype=torch.int64, device=dev)
lib.gift_scan_experiment(expbits)
for i in range(3):
    run.score(fif.dev, q, w.ma, nat.SIM_GAUSSIAN, 0.5, cand_k=4, dense=False, scan_events=ev)
torch.cuda.synchronize()
print(f"{name} scan {ev[0].elapsed_time(ev[1]):.3f} ms (untraced)")
lib.gift_scan_trace(ctypes.c_void_p(TR.data_ptr()))
run.score(fif.dev, q, w.ma, nat.SIM_GAUSSIAN, 0.5, cand_k=4, dense=False, scan_events=ev)
torch.cuda.synchronize()
lib.gift_scan_trace(ctypes.c_void_p(0))
print(f"{name} scan {ev[0].elapsed_time(ev[1]):.3f} ms (traced)")
t2 = TR.view(2, 8, 512, 16).cpu().numpy()
t = t2[kern]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.save(os.path.join(ROOT, "gpurun_out", f"trace_{name}_{drain}_{expbits}.npy"), t2)
names = ["sched", "prod_take", "prod_end", "mma_take", "mma_end", "epi_take", "epi_drained",
         "epi_tail"]
for b in range(2):
    tb = t[b]
    n = int((tb[:, 1] > 0).sum())
    base = tb[0, 0]
    print(f"cta {b}: {n} items")
    for j in range(min(n, 40)):
        row = " ".join(f"{(tb[j, f] - base) if tb[j, f] else -1:9d}" for f in range(8))
        print(f"  {j:3d} N={tb[j, 8]:3d} c={tb[j, 9]:5d} {row}")
    if n > 2:
        d = np.diff(tb[:n, :8].astype(np.float64), axis=0)
        print("  per-item period (median cyc) per stamp:",
              dict(zip(names, np.median(d, axis=0).round(0).tolist())))
        print("  mma busy (end-take) median", np.median(tb[:n, 4] - tb[:n, 3]),
              " epi drain (drained-take)", np.median(tb[:n, 6] - tb[:n, 5]),
              " tail (tail-drained)", np.median(tb[:n, 7] - tb[:n, 6]),
              " prod (end-take)", np.median(tb[:n, 2] - tb[:n, 1]))
        if tb[:n, 12].any():
            print("  tail parts: stage+bar", np.median(tb[:n, 10] - tb[:n, 6]),
                  " masks+bar", np.median(tb[:n, 11] - tb[:n, 10]),
                  " row loop", np.median(tb[:n, 12] - tb[:n, 11]),
                  " (pass 1", np.median(tb[:n, 13] - tb[:n, 11]), ")",
                  " final bar", np.median(tb[:n, 7] - tb[:n, 12]))
