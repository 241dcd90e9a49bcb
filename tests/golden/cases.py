"""Deterministic input builders shared by make_golden.py and the tests.

Pure numpy (`default_rng` streams are machine-independent), so the GPU box
regenerates exactly the inputs the committed golden outputs were computed on.
"""

from __future__ import annotations

import numpy as np


def unit_nonneg_rows(rng, n, d):
    """Random unit-norm non-negative f32 rows (like the reference fixtures,
    conftest.py:5-16)."""
    v = rng.random((n, d))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v.astype(np.float32)


def mixture_views(seed, n_shapes, n_views, dim, n_classes, sigma=0.3, mu0=0.0,
                  zero_views=0, n_queries=0):
    """Gaussian-mixture view sets (BASELINE.json config 1 generator, small):
    class means ~ N(mu0, 1); each shape's views = normalize(relu(mean +
    sigma * N(0, 1))); f32.  `zero_views` rows are zeroed at seeded spots.
    The first n_shapes rows are the database, the next n_queries the queries
    (same class means)."""
    rng = np.random.default_rng(seed)
    means = rng.standard_normal((n_classes, dim)) + mu0
    n_shapes = n_shapes + n_queries
    labels = rng.integers(0, n_classes, size=n_shapes)
    x = means[labels][:, None, :] + sigma * rng.standard_normal((n_shapes, n_views, dim))
    x = np.maximum(x, 0.0)
    nrm = np.linalg.norm(x, axis=2, keepdims=True)
    nrm[nrm == 0] = 1.0
    x = (x / nrm).astype(np.float32)
    if zero_views:
        flat = rng.choice(n_shapes * n_views, size=zero_views, replace=False)
        x.reshape(-1, dim)[flat] = 0.0
    return x, labels


def sampled_codebook(views, k, seed):
    """K distinct non-zero DB view rows sampled without replacement (SURVEY.md
    §8(d) 'Codebooks'; stands in for k-means, divergence D3)."""
    rng = np.random.default_rng(seed)
    flat = views.reshape(-1, views.shape[-1])
    nz = np.flatnonzero(flat.any(axis=1))
    pick = rng.choice(nz, size=k, replace=False)
    return flat[np.sort(pick)].astype(np.float32)


def shape_ids(n, prefix="s"):
    width = max(4, len(str(n)))
    return [f"{prefix}{i:0{width}d}" for i in range(n)]


# End-to-end cases: (name, seed, N, V, d, classes, K, ma, k1, k2, n_queries, top_k, zero_views)
E2E_CASES = [
    ("tiny", 11, 24, 6, 16, 4, 5, 2, 4, 2, 6, 10, 3),
    ("small", 12, 120, 8, 32, 8, 12, 2, 6, 3, 10, 20, 0),
    ("c1like", 13, 400, 16, 64, 12, 16, 1, 10, 4, 12, 50, 0),
]

# evaluate_index cases (overlapping classes: retrieval is imperfect):
# (name, seed, N, V, d, classes, K, ma, k1, k2, sigma)
EVAL_CASES = [
    ("noisy", 21, 150, 8, 32, 10, 12, 2, 6, 3, 1.2),
    ("noisy2", 22, 90, 6, 24, 6, 8, 1, 5, 2, 1.6),
]


# BASELINE.json config 1, exactly: N=1,000 shapes x V=64 views x d=256, a
# 40-class isotropic mixture (means ~ N(0, 1), sigma 0.3, ReLU, L2), K=64
# sampled centroids, ma=1, gaussian sigma=0.5 (cosine for the reference
# goldens), S-IF top-10 neighbour sets (k1=10, k2=4), 100 queries, top-50.
C1 = dict(N=1000, V=64, d=256, classes=40, K=64, ma=1, k1=10, k2=4, n_queries=100, top_k=50,
          sigma=0.5, seed=2016)


def c1_inputs():
    """(db [1000, 64, 256] f32, queries [100, 64, 256] f32, centroids, ids)."""
    views, _ = mixture_views(C1["seed"], C1["N"], C1["V"], C1["d"], C1["classes"],
                             n_queries=C1["n_queries"])
    db, qs = views[:C1["N"]], views[C1["N"]:]
    return db, qs, sampled_codebook(db, C1["K"], C1["seed"] + 1), shape_ids(C1["N"])


def kmeans_inputs(name):
    """Seeded training sets for codebook training (codebook.py:64-108):
    (features, k, seed, max_iters)."""
    rng = np.random.default_rng({"mix": 41, "tiny": 42, "dup": 43, "wide": 44}[name])
    if name == "mix":
        x, _ = mixture_views(41, 40, 5, 32, 6, sigma=0.5)
        return x.reshape(-1, 32).astype(np.float64), 8, 7, 50
    if name == "tiny":  # fewer vectors than centers: tiled
        return rng.random((5, 6)), 12, 3, 50
    if name == "dup":  # exact duplicates: zero-distance draws and empty clusters
        base = rng.random((3, 4))
        return base[rng.integers(0, 3, 40)], 6, 11, 20
    if name == "wide":  # d > 128: the pairwise-summed norms recurse
        return unit_nonneg_rows(rng, 150, 300).astype(np.float64), 6, 5, 50
    raise KeyError(name)


KMEANS_CASES = ["mix", "tiny", "dup", "wide"]
