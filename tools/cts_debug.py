"""Tiny compressed-tile-store scan run (debugging aid: compute-sanitizer target)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]
from cases import mixture_views, sampled_codebook, shape_ids  # noqa: E402

from paper_1604_01879_b200 import matching as mt  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402

os.environ.setdefault("GIFT_TC_PAIR", "0")
views, _ = mixture_views(77, 40, 8, 256, 5, mu0=-0.26, n_queries=2)
db, qs = views[:40], views[40:]
C = sampled_codebook(db, 8, 4)
fif = mt.build_fif_from_tensor(torch.from_numpy(db).cuda(), Codebook(C), shape_ids(40))
print("cts", None if fif.dev.cts is None else fif.dev.cts.numel(), "T", fif.dev.T)
out = {}
for m in ("1", "0"):
    os.environ["GIFT_CTS"] = m
    out[m] = mt.query_fif_batch(fif, qs, 2, "gaussian").cpu().numpy()
    torch.cuda.synchronize()
print("max abs diff", float(np.abs(out["1"] - out["0"]).max()))
