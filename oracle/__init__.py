"""CPU oracle for the GIFT F-IF + S-IF query path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy (and one C helper), the algorithm of the
reference package `shapesearch` (`/root/reference/pkg/src/shapesearch`) for
the hot path named in BASELINE.json: quantize -> F-IF build -> F-IF score ->
top-k -> S-IF build / re-rank.  Every function cites the reference file:line it
follows.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import it, and only as the checker or the timed CPU
baseline.  The product path (`paper_1604_01879_b200`) never imports it and has
no CPU fallback.

Parity pinning: the cosine-mode functions are pinned against golden vectors
produced by the reference itself (`tests/golden/make_golden.py`, checked by
`tests/test_oracle_golden.py`).  The Gaussian-kernel mode (BASELINE.json
north_star; no reference counterpart, SURVEY.md divergence D1) is a
restatement of `query_fif` with the similarity substituted and is pinned only
through the reference's properties (degeneracy, lower bound, monotonicity) —
"parity unpinned" for its absolute values.
"""

from .reference_port import *  # noqa: F401,F403
