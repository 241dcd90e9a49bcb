"""shapesearch.matching on the B200 path (paper_1604_01879_b200.matching)."""
from paper_1604_01879_b200.matching import *  # noqa: F401,F403
from paper_1604_01879_b200 import matching as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})
from .codebook import quantize  # noqa: E402,F401  (re-exported by the reference module)
