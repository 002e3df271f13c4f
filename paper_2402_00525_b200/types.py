"""Host-side mirror of the reference's public types for the render path.

Names, fields, defaults and error behaviour follow the reference package:

* ``Gaussian3D`` / ``Camera``       scene_io.py:52-129
* ``Hierarchical``                   rasterizer.py:70-87
* ``validate_mode`` / ``parse_mode`` rasterizer.py:93-146
* ``RenderConfig``                   rasterizer.py:170-208
* ``TileBin`` / ``PixelRecords`` / ``FrameOutput``  rasterizer.py:215-255
* ``SceneFormatError`` / ``ConfigError`` / ``DataError``  errors.py:4-13

Every reference sort mode runs on the B200 path: ``Hierarchical`` (the
paper's pipeline, the benchmarked hot path), ``GlobalZ`` (the 3DGS order),
``FullPerPixel`` (the exact per-pixel order; the default of ``render`` as in
the reference) and ``Window(size)``.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

SH_COEFFS = 16
TILE_SIZE = 16
OPACITY_EPS = 1.0 / 255.0
NEAR_PLANE = 0.2
GUARD_BAND = 1.3
DILATION = 0.3
INV_SCALE_CLAMP = 1e3


class SceneFormatError(ValueError):
    """A scene or camera violates its format (errors.py:4-5)."""


class ConfigError(ValueError):
    """A run configuration is malformed (errors.py:8-9)."""


class DataError(RuntimeError):
    """Input data passed validation but failed during processing (errors.py:12-13)."""


@dataclass
class Gaussian3D:
    """One anisotropic 3D Gaussian (scene_io.py:52-81): quaternion w,x,y,z;
    linear per-axis scales; linear opacity; SH coefficients [16, 3]."""

    mean: np.ndarray
    rotation: np.ndarray
    scale: np.ndarray
    opacity: float
    sh: np.ndarray

    def __post_init__(self):
        self.mean = np.asarray(self.mean, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(4)
        self.scale = np.asarray(self.scale, dtype=np.float64).reshape(3)
        self.opacity = float(self.opacity)
        self.sh = np.asarray(self.sh, dtype=np.float64).reshape(SH_COEFFS, 3)


@dataclass
class Camera:
    """Pinhole camera with a world->view rotation (scene_io.py:84-129)."""

    rotation: np.ndarray
    position: np.ndarray
    fx: float
    fy: float
    width: int
    height: int
    cx: float | None = None
    cy: float | None = None

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        self.position = np.asarray(self.position, dtype=np.float64).reshape(3)
        self.fx = float(self.fx)
        self.fy = float(self.fy)
        self.width = int(self.width)
        self.height = int(self.height)
        if self.width <= 0 or self.height <= 0:
            raise SceneFormatError("camera image size must be positive")
        if self.fx <= 0 or self.fy <= 0:
            raise SceneFormatError("camera focal lengths must be positive")
        if self.cx is None:
            self.cx = self.width / 2.0
        if self.cy is None:
            self.cy = self.height / 2.0
        self.cx = float(self.cx)
        self.cy = float(self.cy)
        drift = np.abs(self.rotation @ self.rotation.T - np.eye(3)).max()
        if drift > 1e-6:
            raise SceneFormatError(
                f"camera rotation is not orthonormal (residual {drift:.3g})")

    @property
    def view_direction(self) -> np.ndarray:
        return self.rotation[2].copy()


@dataclass(frozen=True)
class GlobalZ:
    """One view-space z key per splat, the 3DGS order (rasterizer.py:48-50);
    K6 = k_render_globalz."""


@dataclass(frozen=True)
class FullPerPixel:
    """The exact per-pixel order (rasterizer.py:53-55); K6 =
    k_render_window (repeated top-48 selection with a shared-memory heap)."""


@dataclass(frozen=True)
class Window:
    """Per-pixel resorting window over the per-tile key stream
    (rasterizer.py:58-67); K6 = k_render_window (a per-pixel shared-memory
    min-heap, sizes up to 512)."""

    size: int = 8


@dataclass(frozen=True)
class Hierarchical:
    """Three-level queue pipeline over 4x4 and 2x2 sub-tiles (rasterizer.py:70-87)."""

    queue_tail: int = 64
    queue_mid: int = 8
    queue_head: int = 4
    batch_load: int = 32
    batch_mid: int = 16
    batch_head: int = 4
    mid_depth_at_center: bool = False


SortMode = GlobalZ | FullPerPixel | Window | Hierarchical


def validate_mode(mode) -> None:
    """rasterizer.py:93-117 (same messages)."""
    if isinstance(mode, Window) or type(mode).__name__ == "Window":
        if mode.size < 1:
            raise ConfigError(f"window size must be >= 1, got {mode.size}")
    elif _is_hier(mode):
        if mode.queue_tail < 64 or mode.queue_tail % 32 != 0:
            raise ConfigError(
                f"tail queue must be a multiple of 32 and at least 64,"
                f" got {mode.queue_tail}")
        if mode.queue_mid < 4 or mode.queue_mid % 4 != 0:
            raise ConfigError(
                f"mid queue must be a positive multiple of 4, got {mode.queue_mid}")
        if mode.queue_head < 1:
            raise ConfigError(f"head queue must hold at least 1, got {mode.queue_head}")
        if mode.batch_load < 1 or mode.batch_load >= mode.queue_tail:
            raise ConfigError("load batch must be positive and below the tail queue")
        if mode.batch_mid < 1 or mode.batch_head < 1:
            raise ConfigError("batch sizes must be positive")
        if mode.batch_head > mode.queue_mid:
            raise ConfigError("head batch cannot exceed the mid queue size")
    elif type(mode).__name__ not in ("GlobalZ", "FullPerPixel"):
        raise ConfigError(f"unknown sort mode {mode!r}")


def _is_hier(mode) -> bool:
    return isinstance(mode, Hierarchical) or type(mode).__name__ == "Hierarchical"


def parse_mode(text: str):
    """rasterizer.py:120-146."""
    t = text.strip().lower().replace("(", ":").rstrip(")")
    if t in ("globalz", "global-z", "global"):
        return GlobalZ()
    if t in ("full", "full-per-pixel", "fullperpixel"):
        return FullPerPixel()
    if t.startswith("window"):
        try:
            size = int(t.split(":", 1)[1])
        except (IndexError, ValueError) as exc:
            raise ConfigError(f"cannot parse window size from {text!r}") from exc
        mode = Window(size)
        validate_mode(mode)
        return mode
    if t.startswith(("hier", "hierarchical")):
        if ":" in t:
            try:
                tail, mid, head = (int(v) for v in t.split(":", 1)[1].split("/"))
            except ValueError as exc:
                raise ConfigError(f"cannot parse queue sizes from {text!r}") from exc
            mode = Hierarchical(queue_tail=tail, queue_mid=mid, queue_head=head)
        else:
            mode = Hierarchical()
        validate_mode(mode)
        return mode
    raise ConfigError(f"unknown sort mode {text!r}")


def mode_name(mode) -> str:
    """rasterizer.py:149-156."""
    n = type(mode).__name__
    if n == "GlobalZ":
        return "globalz"
    if n == "FullPerPixel":
        return "full"
    if n == "Window":
        return f"window:{mode.size}"
    return f"hierarchical:{mode.queue_tail}/{mode.queue_mid}/{mode.queue_head}"


def _default_workers() -> int:
    try:
        return max(1, int(os.environ.get("SPLATSORT_WORKERS", "1")))
    except ValueError:
        return 1


@dataclass
class RenderConfig:
    """rasterizer.py:170-208.  ``workers`` is accepted for compatibility (the
    GPU path is deterministic for any value)."""

    tile_size: int = TILE_SIZE
    opacity_eps: float = OPACITY_EPS
    termination: float = 1e-4
    alpha_cap: float = 0.99
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    near: float = NEAR_PLANE
    guard_band: float = GUARD_BAND
    dilation: float = DILATION
    inv_scale_clamp: float = INV_SCALE_CLAMP
    capture_records: bool = False
    with_depth: bool = False
    workers: int = field(default_factory=_default_workers)
    exact_tile_culling: bool | None = None

    def __post_init__(self):
        self.background = np.asarray(self.background, dtype=np.float64).reshape(3)
        if self.tile_size < 4 or self.tile_size % 4 != 0:
            raise ConfigError("tile size must be a multiple of 4 and at least 4")
        if self.workers < 1:
            raise ConfigError("worker count must be at least 1")
        if not 0 < self.alpha_cap < 1:
            raise ConfigError("alpha cap must lie in (0, 1)")

    def exact_culling(self, mode) -> bool:
        if self.exact_tile_culling is None:
            return type(mode).__name__ != "GlobalZ"
        return self.exact_tile_culling


@dataclass
class SplatBatch:
    """Projected splats of one camera in SoA form (gaussian_math.py:260-307);
    ``render`` accepts one in place of Gaussians and skips projection
    (rasterizer.py:616-618).  conic = (a, b, c); inv_cov3 packed
    (m00, m11, m22, m01, m02, m12); the batch index is the rank."""

    mean2d: np.ndarray
    conic: np.ndarray
    color: np.ndarray
    opacity: np.ndarray
    radius: np.ndarray
    global_depth: np.ndarray
    inv_cov3: np.ndarray
    inv_cov_center: np.ndarray
    mean3d: np.ndarray
    center_dist: np.ndarray
    source_index: np.ndarray

    def __len__(self) -> int:
        return len(self.opacity)


@dataclass
class TileBin:
    """rasterizer.py:215-231."""

    tile_x: int
    tile_y: int
    splat: np.ndarray
    key: np.ndarray

    def __len__(self) -> int:
        return len(self.splat)


@dataclass
class PixelRecords:
    """rasterizer.py:234-243."""

    splat: np.ndarray
    depth: np.ndarray
    alpha: np.ndarray

    def __len__(self) -> int:
        return len(self.splat)


@dataclass
class FrameOutput:
    """rasterizer.py:246-255.  Arrays are float64 numpy (as the reference) unless
    ``render(..., device_output=True)`` asked for the float32 device tensors."""

    color: object
    transmittance: object
    depth: object | None = None
    records: list | None = None
    source_index: object | None = None
    stats: dict = field(default_factory=dict)
    # per-pixel sort error delta (metrics.py:46-73), when rendered with
    # sort_error=True: computed on the GPU during the blend, no records needed
    sort_error: object | None = None
