"""Scan error vs the f64 oracle as a function of the D1 drain interval
(GIFT_FIF_DRAIN_KB), and the scan time: config-4 storage (fp16, fp16-exact
queries, Zipf cells; reduced N) and config-2 storage (f32 planes)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import scale  # noqa: E402
from paper_1604_01879_b200 import matching as mt  # noqa: E402
from paper_1604_01879_b200 import synth  # noqa: E402
from paper_1604_01879_b200.codebook import Codebook  # noqa: E402

dev = torch.device("cuda", 0)
out = []


def run(name, db, qs, C, ma, nq):
    ids = synth.shape_ids(db.shape[0])
    fif = mt.build_fif_from_tensor(db, Codebook(C), ids)
    d = fif.dev
    cell_off, post_ord = d.cell_off.cpu().numpy(), d.post_ord.cpu().numpy()
    feat = d.feat.float().cpu().numpy()
    q = qs[:nq].contiguous()
    qh = q.cpu().numpy()
    cells = scale.quantize_many_mt(C, qh.reshape(-1, qh.shape[2]), ma).reshape(nq, -1, ma)
    ref = scale.fif_scores_many(cell_off, post_ord, lambda a, b: feat[a:b],
                                qh, cells, db.shape[0], "gaussian", 0.5)
    for kb, raw in [(k, r) for k in (1, 2, 4, 8, 16) for r in (True, False)]:
        d.set_variant(drain_kb=kb, raw_accum=raw)
        got = mt.query_fif_batch(fif, q, ma, "gaussian").cpu().numpy()
        m = ref > 0
        sr = (got[m] - ref[m]) / ref[m]
        r = np.abs(sr)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            mt.query_fif_batch(fif, q, ma, "gaussian")
        torch.cuda.synchronize()
        line = {"case": name, "drain_kb": kb, "compensated": not raw, "n": int(m.sum()), "max": float(r.max()),
                "p9999": float(np.quantile(r, 0.9999)), "p99": float(np.quantile(r, 0.99)),
                "mean_signed": float(sr.mean()), "std_signed": float(sr.std()),
                "frac_negative": float((sr < 0).mean()),
                "ms_per_batch": (time.perf_counter() - t0) / 5 * 1000}
        print(json.dumps(line), flush=True)
        out.append(line)
    d.set_variant()
    del fif


w = synth.WORKLOADS["c4s"]
db, qs, Ct = synth.zipf_mixture(w, 20160407, dev)
run("c4s_fp16", db, qs, Ct.cpu().numpy(), 1, 512)
del db, qs
torch.cuda.empty_cache()
w2 = synth.Workload("c2s", 2000, 64, 4096, 55, 256, 2, 0.5, 10, 4, 100, 64, 64, -0.26)
db, qs, _ = synth.mixture(w2, 20160407, dev)
C = synth.sample_centroids(db, 256, 20160408).cpu().numpy()
run("c2s_f32", db, qs, C, 2, 64)
with open(os.path.join(ROOT, "gpurun_out", "drain_error.jsonl"), "w") as fh:
    for line in out:
        fh.write(json.dumps(line) + "\n")
