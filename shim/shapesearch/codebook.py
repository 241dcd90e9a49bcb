"""shapesearch.codebook on the B200 path (paper_1604_01879_b200.codebook)."""
from paper_1604_01879_b200.codebook import *  # noqa: F401,F403
from paper_1604_01879_b200 import codebook as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})
