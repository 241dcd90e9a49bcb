"""B200-native GIFT query path (arXiv 1604.01879): F-IF multi-view matching
followed by S-IF context re-ranking, on hand-written sm_100a kernels
(libgift.so, include/gift.h).

Drop-in for the reference package `shapesearch` on that path: the public API
(`__init__.py:9-29` of the reference) keeps its names and semantics.
"""

from .features import FeatureFile, import_features, write_features
from .index import (
    GraphedQuery,
    IndexBundle,
    IndexConfig,
    build_index,
    build_index_from_feature_file,
    build_index_from_lists,
    build_index_from_views,
    build_index_streamed,
    evaluate_index,
    exact_baseline_report,
    load_bundle,
    query,
    query_batch,
    query_by_id,
    query_many,
    rerank_scores,
    save_bundle,
)

__all__ = [
    "GraphedQuery",
    "FeatureFile",
    "import_features",
    "write_features",
    "IndexBundle",
    "IndexConfig",
    "build_index",
    "build_index_from_feature_file",
    "build_index_from_lists",
    "build_index_from_views",
    "build_index_streamed",
    "evaluate_index",
    "exact_baseline_report",
    "load_bundle",
    "query",
    "query_batch",
    "query_by_id",
    "query_many",
    "rerank_scores",
    "save_bundle",
]

__version__ = "0.1.0"
