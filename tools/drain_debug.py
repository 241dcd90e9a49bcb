"""Which scan variants break at drain intervals > 4 (debug)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from cases import mixture_views, sampled_codebook, shape_ids
from paper_1604_01879_b200 import matching as mt
from paper_1604_01879_b200.codebook import Codebook
dev = torch.device("cuda", 0)
views, _ = mixture_views(5, 600, 20, 1024, 12, n_queries=40)
for storage in ("float16", "float32"):
    db = views[:600].astype(np.float16 if storage == "float16" else np.float32)
    C = sampled_codebook(db.astype(np.float32), 16, 1)
    fif = mt.build_fif_from_tensor(torch.from_numpy(db).to(dev), Codebook(C), shape_ids(600))
    for qname, qs in (("q16", views[600:].astype(np.float16).astype(np.float32)), ("q32", views[600:])):
        for pair in ("off", "on"):
            base = None
            for kb in (1, 4, 8, 16):
                fif.dev.set_variant(pair=pair, drain_kb=kb, raw_accum=True)
                s = mt.query_fif_batch(fif, qs, 1, "gaussian").cpu().numpy()
                if base is None:
                    base = s
                m = base > 0
                err = np.abs(s[m] - base[m]) / base[m]
                print(storage, qname, "pair", pair, "drain", kb, "max rel diff vs drain1 %.2e" % err.max(), flush=True)
    fif.dev.set_variant()
