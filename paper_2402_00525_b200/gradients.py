"""Backward pass of the blended image w.r.t. per-splat screen attributes,
mirroring the reference's ``splatsort.gradients`` (gradients.py:1-162) on the
B200 path: ``backward_render(scene, cam, mode, upstream, cfg)`` returns
``SplatGradients`` (d_color, d_opacity, d_mean2d, d_conic, d_background) in
the projected batch's order.  The GPU replays the forward blend order instead
of storing records (stp_backward in include/stp.h); the chaining stops at
(color, opacity, mean2d, conic) as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .types import DataError, RenderConfig


@dataclass
class SplatGradients:
    """gradients.py:26-49.  d_conic is packed (a, b, c)."""

    d_color: np.ndarray
    d_opacity: np.ndarray
    d_mean2d: np.ndarray
    d_conic: np.ndarray
    d_background: np.ndarray

    @classmethod
    def zeros(cls, n: int) -> "SplatGradients":
        return cls(d_color=np.zeros((n, 3)), d_opacity=np.zeros(n), d_mean2d=np.zeros((n, 2)),
                   d_conic=np.zeros((n, 3)), d_background=np.zeros(3))


def loss_l2(rendered, target):
    """gradients.py:52-67: mean squared error and its gradient."""
    rendered = np.asarray(rendered, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    if rendered.shape != target.shape:
        raise DataError(f"image dims differ: {rendered.shape} vs {target.shape}")
    diff = rendered - target
    return float(np.mean(diff * diff)), 2.0 * diff / diff.size


def backward_render(scene, cam, mode, upstream, cfg: RenderConfig | None = None,
                    device=None) -> SplatGradients:
    """gradients.py:84-104: gradients w.r.t. the projected batch attributes
    for the loss gradient ``upstream`` (H x W x 3) of the rendered image.
    ``scene`` is a Gaussian list / tensor dict (projected by K1) or a
    SplatBatch."""
    from .renderer import Renderer, _require_cuda, _scene_for
    cfg = cfg or RenderConfig()
    dev = _require_cuda(device)
    r = Renderer(scene if hasattr(scene, "mean2d") else _scene_for(scene, dev), mode, cfg, dev)
    return r.backward(cam, upstream)
