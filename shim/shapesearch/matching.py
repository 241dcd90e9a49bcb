"""shapesearch.matching on the B200 path (paper_1604_01879_b200.matching)."""
from paper_1604_01879_b200.matching import *  # noqa: F401,F403
from paper_1604_01879_b200 import matching as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})
from .codebook import quantize  # noqa: E402,F401  (re-exported by the reference module)


def query_fif(fif, query_views, ma: int = DEFAULT_MA, similarity: str = "cosine",
              sigma: float = 0.5, precision: str = "f64"):
    """matching.py:136-161 with the reference's own f64 arithmetic: the shim's
    per-query `query_fif` runs libgift's f64 CUDA-core scan (scores equal the
    reference's to f64 rounding, as its tests assert at 1e-9 / 1e-12);
    `precision="tc"` selects the tensor-core scan, which the batched product
    API (`query_batch`, `query_many`, the engine) always uses."""
    return _m.query_fif(fif, query_views, ma, similarity, sigma, precision)
