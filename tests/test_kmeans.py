"""Codebook training: the reference's train_codebook
(codebook.py:48-108) — goldens tests/golden/kmeans.npz from the reference
itself (make_golden.py `golden_kmeans`).  CPU: the oracle restatement and
the host-side replay of numpy's Generator.choice draws against the goldens;
GPU: the device training (gift_kmeans_*) against the same goldens."""

import numpy as np
import pytest

from cases import KMEANS_CASES, kmeans_inputs
from conftest import load_golden


@pytest.mark.parametrize("name", KMEANS_CASES)
def test_oracle_training_matches_reference(name):
    import oracle

    g = load_golden("kmeans.npz")
    x, k, seed, iters = kmeans_inputs(name)
    np.testing.assert_array_equal(oracle.train_codebook(x, k, seed, iters), g[f"{name}_centroids"])


def test_choice_replay_consumes_the_same_stream():
    """train_codebook replays rng.choice(n, p=p) as cdf = cumsum(p) / cdf[-1],
    searchsorted(rng.random(), 'right'): same index, same stream position."""
    for seed in range(20):
        r = np.random.default_rng(seed)
        n = int(r.integers(1, 200))
        w = r.random(n) ** 3
        w[r.random(n) < 0.3] = 0.0
        if w.sum() == 0:
            w[0] = 1.0
        p = w / w.sum()
        a, b = np.random.default_rng(seed + 100), np.random.default_rng(seed + 100)
        for _ in range(5):
            want = int(a.choice(n, p=p))
            cdf = p.cumsum()
            cdf /= cdf[-1]
            got = int(cdf.searchsorted(b.random(), side="right"))
            assert got == want
        assert a.random() == b.random()


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in KMEANS_CASES if n != "dup"])
def test_device_training_matches_reference(name):
    from paper_1604_01879_b200.codebook import train_codebook

    g = load_golden("kmeans.npz")
    x, k, seed, iters = kmeans_inputs(name)
    cb = train_codebook(x, k, seed=seed, max_iters=iters, channel="A")
    assert cb.centroids.dtype == np.float32 and cb.k == k and cb.channel == "A"
    np.testing.assert_array_equal(cb.centroids, g[f"{name}_centroids"])


@pytest.mark.gpu
def test_device_training_on_duplicates():
    """Exact duplicates: the reference's D^2 to an already chosen point is its
    own rounding noise (|x|^2 - 2 x.c + |c|^2 in BLAS order, ~1e-16), and its
    k-means++ draws then follow that noise, so no other summation order can
    reproduce them (a documented divergence).  The device result must still be
    a Lloyd fixed point made of training points, with every distinct point a
    centroid once k exceeds their count."""
    from paper_1604_01879_b200.codebook import train_codebook

    x, k, seed, iters = kmeans_inputs("dup")
    cb = train_codebook(x, k, seed=seed, max_iters=iters)
    pts = {tuple(r) for r in x.astype(np.float32)}
    assert all(tuple(c) in pts for c in cb.centroids)
    assert {tuple(c) for c in cb.centroids} == pts


@pytest.mark.gpu
def test_device_training_errors():
    from paper_1604_01879_b200.codebook import train_codebook
    from paper_1604_01879_b200.errors import EmptyInput

    with pytest.raises(EmptyInput):
        train_codebook(np.zeros((0, 4)), 3)
    with pytest.raises(EmptyInput):
        train_codebook(np.zeros(5), 3)
