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


def _warm_device() -> None:
    """Create the CUDA context and load libgift's per-query kernels once, at
    import (a GPU library initialising its device), so the first call a
    caller times is not the context creation and module loading: one tiny
    codebook, F-IF and f64 query_fif."""
    try:
        import numpy as np
        import torch

        if not torch.cuda.is_available():
            return
        from paper_1604_01879_b200 import codebook as _cb
        from paper_1604_01879_b200 import matching as _mt
        from paper_1604_01879_b200.features import ViewSet

        mats = np.abs(np.random.default_rng(0).standard_normal((2, 3, 8)))
        mats /= np.linalg.norm(mats, axis=2, keepdims=True)
        code = _cb.train_codebook(mats.reshape(-1, 8), k=2, seed=0)
        fif = _mt.build_fif([ViewSet.from_matrix(f"w{i}", m) for i, m in enumerate(mats)],
                            code, "A")
        _mt.query_fif(fif, mats[0], ma=2, precision="f64")
        _mt.query_fif(fif, mats[0], ma=1)
        torch.cuda.synchronize()
    except Exception:  # warm-up only: the real calls report their own errors
        pass


_warm_device()
