"""shapesearch.features: view containers and GIFTFT1 ingress on the B200 path
(paper_1604_01879_b200.features); the depth descriptors (features.py:74-118,
outside the GPU path) are the reference's, returning this module's
ViewDescriptor."""
from paper_1604_01879_b200.features import *  # noqa: F401,F403
from paper_1604_01879_b200 import features as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})

DEFAULT_GRID = 8
DEFAULT_CELLS = 4
DEFAULT_BINS = 8


def _ref():
    from ._ref import load

    return load("features_ref")


def extract_grid_descriptor(image, grid: int = DEFAULT_GRID, channel: str = "A"):
    d = _ref().extract_grid_descriptor(image, grid, channel=channel)
    return ViewDescriptor(values=d.values, channel=d.channel)  # noqa: F405


def extract_gradient_descriptor(image, cells: int = DEFAULT_CELLS, bins: int = DEFAULT_BINS,
                                channel: str = "B"):
    d = _ref().extract_gradient_descriptor(image, cells, bins, channel=channel)
    return ViewDescriptor(values=d.values, channel=d.channel)  # noqa: F405
