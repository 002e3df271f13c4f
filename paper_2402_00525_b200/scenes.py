"""Deterministic synthetic scenes for parity tests and the benchmark.

All generators return float32 SoA arrays in the drop-in layout
(``means[N,3]``, ``quats[N,4]`` w,x,y,z, ``scales[N,3]``, ``opacity[N]``,
``sh[N,K,3]``) plus ``Camera`` objects.  Inputs are float32 so the B200 path
and the float64 CPU oracle consume identical values.

* ``random_cloud``   restates the reference fixture (fixtures.py:191-235) with
  the same ``numpy.random.default_rng`` call sequence, so config #1 can be
  rebuilt where the reference package is absent (the GPU box).
* ``config_scene``   the BASELINE.json configs C1..C5 as calibrated in
  SURVEY.md section 8(d).
"""

from __future__ import annotations

import math

import numpy as np

from .types import Camera

_SH0 = 0.28209479177387814


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def random_cloud_arrays(n: int = 100, seed: int = 0):
    """fixtures.py:191-217 (same rng call order), as float64 arrays."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(1.8, 4.5, n)
    x = rng.uniform(-0.25, 0.25, n) * z
    y = rng.uniform(-0.25, 0.25, n) * z
    scales = np.exp(rng.uniform(np.log(0.04), np.log(0.22), (n, 3)))
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opacity = rng.uniform(0.15, 0.6, n)
    rgb = rng.uniform(0.05, 0.95, (n, 3))
    rest = rng.uniform(-0.04, 0.04, (n, 15, 3))
    sh = np.zeros((n, 16, 3))
    sh[:, 0] = (rgb - 0.5) / _SH0
    sh[:, 1:] = rest
    means = np.stack([x, y, z], axis=1)
    return {"means": means, "quats": quats, "scales": scales, "opacity": opacity, "sh": sh}


def random_cloud_cameras():
    """fixtures.py:218-235."""
    phi = np.deg2rad(3.0)
    c, s = np.cos(phi), np.sin(phi)
    roty = np.array([[c, 0.0, -s], [0.0, 1.0, 0.0], [s, 0.0, c]])
    return [
        Camera(rotation=np.eye(3), position=np.zeros(3), fx=110.0, fy=110.0, width=128, height=128),
        Camera(rotation=roty, position=np.zeros(3), fx=110.0, fy=110.0, width=128, height=128),
    ]


def to_f32_scene(arrs: dict) -> dict:
    return {k: _f32(v) for k, v in arrs.items()}


def look_at(position, target, up=(0.0, -1.0, 0.0)) -> np.ndarray:
    """World->view rotation (rows = view axes x right, y down, z forward)."""
    p = np.asarray(position, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - p
    f /= np.linalg.norm(f)
    u = np.asarray(up, dtype=np.float64)
    r = np.cross(f, u)
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f])
    # re-orthonormalise to well below the Camera 1e-6 check
    uu, _, vt = np.linalg.svd(R)
    return uu @ vt


def _common_attrs(rng, n, sh_coeffs=16, scale_lo=0.003, scale_hi=0.03):
    scales = np.exp(rng.uniform(np.log(scale_lo), np.log(scale_hi), (n, 3)))
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opacity = rng.uniform(0.05, 0.99, n)
    sh = rng.normal(0.0, 0.2, (n, sh_coeffs, 3))
    return scales, quats, opacity, sh


def frustum_cloud(n, seed, width, height, f, z_lo=2.0, z_hi=12.0, sh_coeffs=16,
                  elongated_frac=0.0):
    """C2/C4 law: means uniform in a 1.1x frustum, depth
    U(z_lo, z_hi), log-uniform scales [0.003, 0.03], N(0,.2^2) SH."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(z_lo, z_hi, n)
    x = rng.uniform(-1, 1, n) * 1.1 * z * width / (2 * f)
    y = rng.uniform(-1, 1, n) * 1.1 * z * height / (2 * f)
    scales, quats, opacity, sh = _common_attrs(rng, n, sh_coeffs)
    if elongated_frac > 0:
        m = rng.random(n) < elongated_frac
        scales[m] = np.array([0.7, 0.02, 0.02])
    return {"means": np.stack([x, y, z], 1), "quats": quats, "scales": scales,
            "opacity": opacity, "sh": sh}


def garden_scene(n, seed, density=1.0):
    """C3/C5: a Mip-NeRF-360-garden-like layout (y is down): a ground disc, a
    central object cluster on a table-height plinth and a far backdrop shell.
    ``density`` < 1 thins the cloud and widens splats (the paper's Opacity
    Decay statistics)."""
    rng = np.random.default_rng(seed)
    n_ground = int(0.50 * n)
    n_obj = int(0.22 * n)
    n_back = n - n_ground - n_obj
    r = 12.0 * np.sqrt(rng.random(n_ground))
    th = rng.random(n_ground) * 2 * np.pi
    ground = np.stack([r * np.cos(th), 1.0 + rng.normal(0, 0.06, n_ground), r * np.sin(th)], 1)
    obj = rng.normal(0, 1, (n_obj, 3)) * np.array([1.0, 0.6, 1.0]) + np.array([0, 0.1, 0])
    rb = rng.uniform(10.0, 14.0, n_back)
    thb = rng.random(n_back) * 2 * np.pi
    yb = rng.uniform(-3.0, 1.0, n_back)
    back = np.stack([rb * np.cos(thb), yb, rb * np.sin(thb)], 1)
    means = np.concatenate([ground, obj, back])
    widen = 1.0 / math.sqrt(max(density, 1e-3))
    scales, quats, opacity, sh = _common_attrs(rng, n, 16, 0.003 * widen, 0.03 * widen)
    scales[n_ground + n_obj:] *= 4.0   # backdrop splats are far and large
    perm = rng.permutation(n)
    return {"means": means[perm], "quats": quats[perm], "scales": scales[perm],
            "opacity": opacity[perm], "sh": sh[perm]}


def orbit_cameras(n_views, radius=4.0, height=-1.2, target=(0.0, 0.3, 0.0), width=1920,
                  height_px=1080, f=1100.0, yaw0=0.0, yaw_span=2 * np.pi):
    cams = []
    for v in range(n_views):
        yaw = yaw0 + yaw_span * v / n_views
        pos = np.array([radius * np.sin(yaw), height, -radius * np.cos(yaw)])
        cams.append(Camera(rotation=look_at(pos, target), position=pos, fx=f, fy=f,
                           width=width, height=height_px))
    return cams


def yaw_sweep_cameras(n_views, position=(0.0, -1.2, -4.0), target=(0.0, 0.3, 0.0),
                      half_span_deg=15.0, width=1920, height_px=1080, f=1100.0):
    """C5: a camera at a FIXED position panning its yaw
    over +-half_span around the view of ``target`` (a rotation sweep, cf. the
    popping pan fixtures.py:54-62,144-156).  Frame v's forward axis is the
    base forward rotated about the world vertical (y) axis."""
    base = look_at(position, target)
    cams = []
    for v in range(n_views):
        a = np.deg2rad(-half_span_deg + 2 * half_span_deg * v / max(n_views - 1, 1))
        c, s_ = np.cos(a), np.sin(a)
        ry = np.array([[c, 0.0, s_], [0.0, 1.0, 0.0], [-s_, 0.0, c]])  # world-frame yaw
        R = base @ ry.T          # world->view of the yawed camera (view axes rotated by ry)
        uu, _, vt = np.linalg.svd(R)
        cams.append(Camera(rotation=uu @ vt, position=np.asarray(position, dtype=np.float64),
                           fx=f, fy=f, width=width, height=height_px))
    return cams


CONFIGS = {
    "C1": "synthetic 10k random Gaussians, SH degree 0, single 256x256 view",
    "C2": "synthetic 1M Gaussians, SH degree 3, single 1920x1080 view",
    "C3": "synthetic 3M-Gaussian garden-scale scene, 256-view 1080p orbit",
    "C4": "synthetic 6M Gaussians at 3840x2160 (culling and queue stress)",
    "C5": "synthetic 1.5M half-density scene, 1080p rotation sweep",
}


def config_cameras(name: str, n_views: int | None = None):
    """Cameras of a config without generating its scene."""
    name = name.upper()
    if name == "C3":
        return orbit_cameras(n_views or 256)
    if name == "C5":
        return yaw_sweep_cameras(n_views or 240)
    return config_scene(name, n=16, n_views=n_views)[1]


def config_scene(name: str, n: int | None = None, n_views: int | None = None):
    """(scene f32 arrays, cameras) for BASELINE.json configs C1..C5.
    ``n`` / ``n_views`` override the size for scaled-down parity runs."""
    name = name.upper()
    if name == "C1":
        arrs = random_cloud_arrays(n or 10000, 0)
        arrs["sh"] = arrs["sh"][:, :1]          # SH degree 0 (sh[1:] = 0)
        cam = Camera(rotation=np.eye(3), position=np.zeros(3), fx=220.0, fy=220.0,
                     width=256, height=256)
        return to_f32_scene(arrs), [cam]
    if name == "C2":
        arrs = frustum_cloud(n or 1_000_000, 1, 1920, 1080, 1100.0)
        cam = Camera(rotation=np.eye(3), position=np.zeros(3), fx=1100.0, fy=1100.0,
                     width=1920, height=1080)
        return to_f32_scene(arrs), [cam]
    if name == "C3":
        arrs = garden_scene(n or 3_000_000, 3)
        return to_f32_scene(arrs), orbit_cameras(n_views or 256)
    if name == "C4":
        arrs = frustum_cloud(n or 6_000_000, 4, 3840, 2160, 2200.0, z_lo=2.0, z_hi=6.0,
                             elongated_frac=0.02)
        cam = Camera(rotation=np.eye(3), position=np.zeros(3), fx=2200.0, fy=2200.0,
                     width=3840, height=2160)
        return to_f32_scene(arrs), [cam]
    if name == "C5":
        arrs = garden_scene(n or 1_500_000, 5, density=0.5)
        return to_f32_scene(arrs), yaw_sweep_cameras(n_views or 240)
    raise KeyError(name)
