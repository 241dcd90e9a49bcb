"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every scan variant, the reduces, top-k, activations, S-IF."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from cases import mixture_views, sampled_codebook, shape_ids
import paper_1604_01879_b200 as gift
from paper_1604_01879_b200 import matching as mt
from paper_1604_01879_b200.codebook import Codebook
dev = torch.device("cuda", 0)
views, _ = mixture_views(7, 300, 8, 256, 6, n_queries=40)
for storage in ("float16", "float32"):
    db = views[:300].astype(np.float16 if storage == "float16" else np.float32)
    C = sampled_codebook(db.astype(np.float32), 5, 1)
    cfg = gift.IndexConfig(n_views=8, codebook_size=5, ma=2, k1=6, k2=3, imported=True,
                           similarity="gaussian", storage_dtype=storage)
    b = gift.build_index_from_views(db, shape_ids(300), cfg,
                                    codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")})
    for q in (views[300:].astype(np.float16).astype(np.float32), views[300:]):
        for pair in ("off", "on"):
            b.fifs["A"].dev.set_variant(pair=pair)
            gift.query_batch(b, q, top_k=20)
    b.fifs["A"].dev.set_variant()
# ma = 1, fp16 storage, many queries: dense cells (probe-major scan) and the
# owner reduce with its single-segment fast kernel (forced by the flag)
v1, _ = mixture_views(9, 400, 8, 64, 4, n_queries=120)
db = v1[:400].astype(np.float16)
C = sampled_codebook(db.astype(np.float32), 3, 2)
cfg = gift.IndexConfig(n_views=8, codebook_size=3, ma=1, k1=6, k2=3, imported=True,
                       similarity="gaussian", storage_dtype="float16")
b = gift.build_index_from_views(db, shape_ids(400), cfg,
                                codebooks={"A": Codebook(C, "A"), "B": Codebook(C, "B")})
q16 = v1[400:].astype(np.float16).astype(np.float32)
for red in ("auto", "owner"):
    b.fifs["A"].dev.set_variant(reduce=red)
    gift.query_batch(b, q16, top_k=20)
b.fifs["A"].dev.set_variant()
torch.cuda.synchronize()
print("sanitize workload done")
