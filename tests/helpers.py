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
