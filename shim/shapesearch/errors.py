"""shapesearch.errors: the B200 package's hierarchy (same classes as
errors.py:4-69)."""
from paper_1604_01879_b200.errors import *  # noqa: F401,F403
from paper_1604_01879_b200.errors import ShapeSearchError  # noqa: F401
