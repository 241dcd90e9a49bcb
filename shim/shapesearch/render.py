"""shapesearch.render: the reference's own module (outside the GPU path),
re-exported with its in-scope imports pointed at this shim."""
from ._ref import reexport

reexport(globals(), "render")
