"""shapesearch.rerank on the B200 path (paper_1604_01879_b200.rerank)."""
from paper_1604_01879_b200.rerank import *  # noqa: F401,F403
from paper_1604_01879_b200 import rerank as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})
