"""Host-side API surface (CPU): config validation and error mapping."""

import pytest

from paper_1604_01879_b200 import IndexConfig, errors
from paper_1604_01879_b200.index import _REFERENCE_FIELDS


def test_config_defaults_match_reference():
    c = IndexConfig()
    assert (c.n_views, c.codebook_size, c.ma, c.k1, c.k2, c.alpha, c.seed) == (64, 256, 2, 10, 4, 0.5, 0)
    assert c.similarity == "cosine" and c.storage_dtype == "float32"
    assert len(_REFERENCE_FIELDS) == 12


@pytest.mark.parametrize("kw", [dict(k1=0), dict(alpha=0.0), dict(ma=300), dict(similarity="l2"),
                                dict(sigma=0.0), dict(storage_dtype="int8")])
def test_config_validation(kw):
    with pytest.raises(ValueError):
        IndexConfig(**kw)


def test_status_mapping():
    assert isinstance(errors.from_status(2, "x"), errors.DimensionMismatch)
    assert isinstance(errors.from_status(3, "x"), errors.EmptySet)
    assert isinstance(errors.from_status(1, "x"), ValueError)
    assert isinstance(errors.from_status(4, "x"), errors.ShapeSearchError)
