"""B200-native hierarchical sorted Gaussian-splatting forward renderer
(StopThePop, arXiv 2402.00525), a drop-in for the reference package's
``render(scene, cam, Hierarchical(), cfg)`` path (and its other sort modes).

Public API mirrors ``splatsort`` (reference __init__.py:42-61) for this path.
Importing the package does not need a GPU; rendering does (no CPU fallback).
"""

from .types import (  # noqa: F401
    Camera, ConfigError, DataError, FrameOutput, FullPerPixel, Gaussian3D, GlobalZ,
    Hierarchical, PixelRecords, RenderConfig, SceneFormatError, SortMode, SplatBatch, TileBin,
    Window,
    mode_name, parse_mode, validate_mode,
)

__all__ = [
    "Camera", "ConfigError", "DataError", "FrameOutput", "FullPerPixel", "Gaussian3D",
    "GlobalZ", "Hierarchical", "PixelRecords", "RenderConfig", "SceneFormatError", "SortMode",
    "SplatBatch",
    "TileBin", "Window", "mode_name", "parse_mode", "validate_mode", "render", "render_depth",
    "render_trajectory", "Renderer", "GaussianScene", "sort_error", "SortErrorStats",
    "backward_render", "SplatGradients", "loss_l2", "load_ply", "load_ply_arrays",
    "load_ply_scene", "load_cameras", "consistency",
]


def __getattr__(name):
    # torch-dependent entry points load lazily
    if name in ("render", "render_depth", "render_trajectory", "Renderer", "GaussianScene",
                "sort_error", "SortErrorStats"):
        from . import renderer
        return getattr(renderer, name)
    if name == "consistency":
        import importlib
        return importlib.import_module(".consistency", __name__)
    if name in ("load_ply", "load_ply_arrays", "load_ply_scene", "load_cameras"):
        from . import scene_io
        return getattr(scene_io, name)
    if name in ("backward_render", "SplatGradients", "loss_l2"):
        from . import gradients
        return getattr(gradients, name)
    raise AttributeError(name)
