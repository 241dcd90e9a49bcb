"""Comparators shared by the parity tests."""

import numpy as np

from conftest import load_golden  # noqa: F401

RTOL = 1e-5  # north_star: similarity scores within 1e-5 relative error


def unpack_acts(g, prefix):
    lens = g[f"{prefix}_len"]
    offs = np.concatenate([[0], np.cumsum(lens)])
    idx, val = g[f"{prefix}_idx"], g[f"{prefix}_val"]
    return [(idx[offs[i]:offs[i + 1]].astype(np.int64), val[offs[i]:offs[i + 1]],
             float(g[f"{prefix}_norm"][i])) for i in range(len(lens))]


def unpack_lists(g, key, lens_key):
    lens = g[lens_key]
    offs = np.concatenate([[0], np.cumsum(lens)])
    arr = g[key]
    return [arr[offs[i]:offs[i + 1]] for i in range(len(lens))]


def assert_ranking_close(got_ids, got_scores, ref_ids, ref_scores, rtol=RTOL, atol=1e-12):
    """Ranked lists identical except for swaps among scores tied within
    rtol (north_star); scores compared position by position."""
    got_ids, ref_ids = list(got_ids), list(ref_ids)
    got_scores = np.asarray(got_scores, dtype=np.float64)
    ref_scores = np.asarray(ref_scores, dtype=np.float64)
    assert len(got_ids) == len(ref_ids)
    np.testing.assert_allclose(got_scores, ref_scores, rtol=rtol, atol=atol)
    tol = lambda a, b: abs(a - b) <= rtol * max(abs(a), abs(b)) + atol  # noqa: E731
    n = len(ref_ids)
    i = 0
    while i < n:
        j = i
        while j + 1 < n and tol(ref_scores[j + 1], ref_scores[i]):
            j += 1
        grp_ref = set(ref_ids[i:j + 1])
        grp_got = set(got_ids[i:j + 1])
        if j + 1 < n:
            assert grp_ref == grp_got, (i, j, ref_ids[i:j + 1], got_ids[i:j + 1])
        else:
            # the last tie group may be cut by top_k: ids must still tie
            for k in range(i, j + 1):
                if got_ids[k] not in grp_ref:
                    assert tol(got_scores[k], ref_scores[i]), (k, got_ids[k])
        i = j + 1


def assert_act_close(got, ref, rtol=RTOL, atol=1e-12):
    gi, gv, gn = got
    ri, rv, rn = ref
    np.testing.assert_array_equal(np.asarray(gi), np.asarray(ri))
    np.testing.assert_allclose(gv, rv, rtol=rtol, atol=atol)
    assert abs(gn - rn) <= rtol * abs(rn) + atol


def rel_err_stats(got, ref):
    """Relative-error summary over the scores the reference makes positive
    (max, p99.99, p99, count), plus how many zero / non-zero patterns differ."""
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    m = ref > 0
    r = np.abs(got[m] - ref[m]) / ref[m] if m.any() else np.zeros(1)
    return {"n": int(m.sum()), "max": float(r.max()), "p9999": float(np.quantile(r, 0.9999)),
            "p99": float(np.quantile(r, 0.99)), "zero_mismatch": int(((got == 0) != (ref == 0)).sum())}


def record_parity(config, check, stats):
    """Append one parity measurement to $GIFT_PARITY_OUT (JSON lines; the GPU
    runs copy it under profiles/) and print it."""
    import json
    import os

    line = {"config": config, "check": check, **stats}
    print("PARITY", json.dumps(line))
    path = os.environ.get("GIFT_PARITY_OUT")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(line) + "\n")


def assert_topk_rows_close(got, ref, rtol=RTOL, atol=1e-12):
    """Top-k activation rows (indices ascending, values): identical supports
    with values within rtol, except members whose scores tie the row's
    boundary (its smallest kept score) within rtol, which may be exchanged
    (north_star: swaps among scores tied within the tolerance).  got/ref:
    lists of (indices, values).  Returns the number of exchanged entries."""
    swaps = 0
    for r, ((gi, gv), (ri, rv)) in enumerate(zip(got, ref)):
        gd = dict(zip(np.asarray(gi).tolist(), np.asarray(gv).tolist()))
        rd = dict(zip(np.asarray(ri).tolist(), np.asarray(rv).tolist()))
        for k in gd.keys() & rd.keys():
            assert abs(gd[k] - rd[k]) <= rtol * abs(rd[k]) + atol, (r, k, gd[k], rd[k])
        diff = (gd.keys() ^ rd.keys())
        if diff:
            edge = min(rd.values())
            for k in diff:
                v = gd.get(k, rd.get(k))
                assert abs(v - edge) <= rtol * abs(edge) + atol, (r, k, v, edge)
            swaps += len(diff)
    return swaps
