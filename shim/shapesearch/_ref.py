"""The reference package's out-of-scope modules (mesh IO, rendering, depth
descriptors, dataset generator, CLI, HTTP service), loaded from a reference
install under the alias package `_shapesearch_ref`.  Their relative imports
of the in-scope modules (errors, features, codebook, matching, rerank,
index, evaluation) resolve to THIS shim, i.e. to the B200 path: the CLI and
the service drive the GPU index, and every exception shares one hierarchy.

Search order for the reference sources: $SHAPESEARCH_REF, baseline/_ref
(a `pip install --target` of the reference), /root/reference/pkg/src.
"""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys
import types

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ALIAS = "_shapesearch_ref"
_SHIMMED = ("errors", "features", "codebook", "matching", "rerank", "index", "evaluation")


def _source_dir():
    for cand in (os.environ.get("SHAPESEARCH_REF"),
                 os.path.join(_ROOT, "baseline", "_ref", "shapesearch"),
                 "/root/reference/pkg/src/shapesearch"):
        if cand and os.path.isfile(os.path.join(cand, "mesh.py")):
            return cand
    return None


def _package():
    pkg = sys.modules.get(ALIAS)
    if pkg is not None:
        return pkg
    src = _source_dir()
    if src is None:
        raise ImportError("the reference's rendering / CLI modules are not installed: set "
                          "SHAPESEARCH_REF or pip-install the reference into baseline/_ref")
    pkg = types.ModuleType(ALIAS)
    pkg.__path__ = [src]
    pkg.__file__ = os.path.join(src, "__init__.py")
    sys.modules[ALIAS] = pkg
    for name in _SHIMMED:  # in-scope modules: this shim (the GPU path)
        sys.modules[f"{ALIAS}.{name}"] = importlib.import_module(f"shapesearch.{name}")
    return pkg


def load(name: str):
    """A reference module by name (mesh, render, dataset, cli, service), or the
    reference's own features module as `features_ref` (depth descriptors)."""
    _package()
    real = name[:-4] if name.endswith("_ref") else name
    full = f"{ALIAS}.{name}"
    mod = sys.modules.get(full)
    if mod is None:
        spec = importlib.util.spec_from_file_location(
            full, os.path.join(_source_dir(), f"{real}.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[full] = mod
        spec.loader.exec_module(mod)
    return mod


def reexport(module_globals: dict, name: str) -> None:
    mod = load(name)
    for k, v in vars(mod).items():
        if not k.startswith("__"):
            module_globals.setdefault(k, v)


def fill_missing(module_globals: dict, name: str, names) -> None:
    """Off-path helpers the B200 module does not restate (report writers):
    taken from the reference's own module `name`."""
    try:
        mod = load(f"{name}_ref") if name != "features" else load("features_ref")
    except ImportError:
        return
    for k in names:
        if k not in module_globals and hasattr(mod, k):
            module_globals[k] = getattr(mod, k)
