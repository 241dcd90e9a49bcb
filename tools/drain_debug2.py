"""c4s: where do drain-8 scores deviate from drain-4 ones (debug)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1604_01879_b200 import matching as mt, synth, engine as eg
from paper_1604_01879_b200.codebook import Codebook
dev = torch.device("cuda", 0)
w = synth.WORKLOADS["c4s"]
db, qs, Ct = synth.zipf_mixture(w, 20160407, dev)
fif = mt.build_fif_from_tensor(db, Codebook(Ct.cpu().numpy()), synth.shape_ids(w.n_shapes))
d = fif.dev
print("P", d.P, "S", d.S, "T", d.T, "seg_len_max", d.seg_len_max, "flags", d.view.flags, flush=True)
for nq in (8, 64, 512):
    q = qs[:nq].contiguous()
    out = {}
    for kb in (4, 8):
        for pair in ("off", "on"):
            d.set_variant(drain_kb=kb, pair=pair, raw_accum=True)
            out[kb, pair] = mt.query_fif_batch(fif, q, 1, "gaussian").cpu().numpy()
    base = out[4, "off"]
    for k, s in out.items():
        m = base > 0
        err = np.abs(s - base)
        bad = np.argwhere(err > 1e-4 * np.maximum(base, 1e-30))
        print(nq, k, "max abs diff %.3e" % err.max(), "n_bad", len(bad), bad[:5].tolist(), flush=True)
cells = eg.quantize_rows(d.cb, qs[:512].reshape(-1, 1024), 1).cpu().numpy().reshape(512, 20)
cnt = np.bincount(cells[cells >= 0].ravel(), minlength=4096)
print("probes per cell max", cnt.max(), "cells probed", (cnt > 0).sum())
