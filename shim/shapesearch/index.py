"""shapesearch.index on the B200 path (paper_1604_01879_b200.index), with the
reference's CPU mesh rendering (index.py:106-139) plugged in front of it, so
mesh manifests and mesh queries work as in the reference."""
from paper_1604_01879_b200.index import *  # noqa: F401,F403
from paper_1604_01879_b200 import index as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})


def compute_viewset(mesh, config):
    """index.py:106-114: render every view of the pose-normalized mesh and
    extract both descriptor channels (the reference's renderer)."""
    from . import features as ft
    from ._ref import load

    render = load("render")
    normalized = load("mesh").normalize_pose(mesh)
    vs = ft.ViewSet(shape_id=mesh.id)
    for camera in render.camera_positions(config.n_views):
        image = render.render_depth(normalized, camera, config.resolution)
        vs.add("A", ft.extract_grid_descriptor(image, config.grid, channel="A"))
        vs.add("B", ft.extract_gradient_descriptor(image, config.cells, config.bins, channel="B"))
    return vs


def _install_renderer():
    try:
        from ._ref import load

        mesh = load("mesh")
    except ImportError:
        return  # no reference install: feature files / view tensors only
    _m.set_renderer(compute_viewset, mesh.load_mesh, mesh.Mesh)


_install_renderer()
