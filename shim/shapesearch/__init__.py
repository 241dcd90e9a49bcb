"""`shapesearch` drop-in shim: the reference package's import surface
(`/root/reference/pkg/src/shapesearch`, `__init__.py:9-29`) served by the
B200 path (`paper_1604_01879_b200`).

In-scope modules (codebook, matching, rerank, index, features, evaluation,
errors) are this package's own; the out-of-scope ones (mesh, render,
dataset, cli, service) are the reference's, re-exported through `_ref` with
their in-scope imports pointed back here.  Put the directory holding this
package first on sys.path to run reference code and tests unchanged."""

from .index import (
    IndexBundle,
    IndexConfig,
    build_index,
    evaluate_index,
    load_bundle,
    query,
    query_by_id,
    save_bundle,
)

__all__ = [
    "IndexBundle",
    "IndexConfig",
    "build_index",
    "evaluate_index",
    "load_bundle",
    "query",
    "query_by_id",
    "save_bundle",
]

__version__ = "0.1.0"
