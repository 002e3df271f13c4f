"""Scene and camera input for the B200 path.

The reference reads 3DGS checkpoints into Python ``Gaussian3D`` objects
(``scene_io.load_ply``, scene_io.py:189-254) and JSON camera arrays
(``load_cameras``, :366-417).  Here a checkpoint is decoded column-wise
straight into the drop-in float32 layout the kernels read (``means[N,3]``,
``quats[N,4]`` w,x,y,z, ``scales[N,3]``, ``opacity[N]``, ``sh[N,16,3]``) and,
with ``load_ply_scene``, uploaded once to the device -- no per-Gaussian Python
objects on the way.  Decoding follows the reference: scales = exp(stored),
opacity = sigmoid(stored), quaternions normalised, f_rest channel-major
(15 red, 15 green, 15 blue coefficients); records that decode to non-finite
or degenerate values raise ``SceneFormatError`` as the reference does.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .types import Camera, Gaussian3D, SceneFormatError

# PLY scalar type names -> little-endian numpy codes
_TYPES = {"char": "i1", "int8": "i1", "uchar": "u1", "uint8": "u1", "short": "<i2",
          "int16": "<i2", "ushort": "<u2", "uint16": "<u2", "int": "<i4", "int32": "<i4",
          "uint": "<u4", "uint32": "<u4", "float": "<f4", "float32": "<f4",
          "double": "<f8", "float64": "<f8"}

_NEED = (["x", "y", "z"] + [f"f_dc_{k}" for k in range(3)] + [f"f_rest_{k}" for k in range(45)]
         + ["opacity"] + [f"scale_{k}" for k in range(3)] + [f"rot_{k}" for k in range(4)])


def _header(raw: bytes):
    """(vertex count, payload offset, numpy record dtype) of a binary PLY."""
    marker = raw.find(b"end_header")
    if marker < 0:
        raise SceneFormatError("PLY header has no end_header")
    nl = raw.find(b"\n", marker)
    if nl < 0:
        raise SceneFormatError("PLY header is not terminated")
    text = raw[:marker].decode("ascii", errors="replace").splitlines()
    if not text or text[0].strip() != "ply":
        raise SceneFormatError("not a PLY file")
    count, fields, element, fmt = None, [], None, None
    for line in text[1:]:
        words = line.split()
        if not words or words[0] in ("comment", "obj_info"):
            continue
        if words[0] == "format":
            fmt = words[1] if len(words) > 1 else ""
        elif words[0] == "element":
            element = words[1]
            if element == "vertex":
                count = int(words[2])
        elif words[0] == "property" and element == "vertex":
            if words[1] == "list":
                raise SceneFormatError("list properties are not supported")
            code = _TYPES.get(words[1])
            if code is None:
                raise SceneFormatError(f"unsupported property type {words[1]!r}")
            fields.append((words[2], code))
    if fmt is None:
        raise SceneFormatError("PLY header missing format line")
    if fmt != "binary_little_endian":
        raise SceneFormatError(f"unsupported PLY format {fmt!r}")
    if count is None:
        raise SceneFormatError("PLY header missing vertex element")
    return count, nl + 1, np.dtype(fields)


def load_ply_arrays(path) -> dict:
    """Decode a 3DGS binary PLY into the drop-in float32 arrays."""
    raw = Path(path).read_bytes()
    n, off, dt = _header(raw)
    missing = [k for k in _NEED if k not in dt.names]
    if missing:
        raise SceneFormatError(f"PLY missing required property {missing[0]!r}")
    if len(raw) - off < n * dt.itemsize:
        raise SceneFormatError(f"PLY payload truncated: need {n * dt.itemsize} bytes, "
                               f"found {len(raw) - off}")
    rec = np.frombuffer(raw, dtype=dt, count=n, offset=off)

    def cols(names):
        return np.stack([np.asarray(rec[k], dtype=np.float64) for k in names], axis=1) \
            if n else np.zeros((0, len(names)))

    means = cols(["x", "y", "z"])
    q = cols([f"rot_{k}" for k in range(4)])
    qn = np.sqrt((q * q).sum(axis=1))
    degenerate_q = qn < 1e-12
    q = q / np.where(degenerate_q, 1.0, qn)[:, None]
    scales = np.exp(cols([f"scale_{k}" for k in range(3)]))
    logit = np.asarray(rec["opacity"], dtype=np.float64) if n else np.zeros(0)
    opacity = 1.0 / (1.0 + np.exp(-logit))
    sh = np.empty((n, 16, 3))
    sh[:, 0, :] = cols([f"f_dc_{k}" for k in range(3)])
    rest = cols([f"f_rest_{k}" for k in range(45)]).reshape(n, 3, 15)  # [rgb][coefficient]
    sh[:, 1:, :] = rest.transpose(0, 2, 1)
    ok = (np.isfinite(means).all(1) & np.isfinite(q).all(1) & ~degenerate_q &
          np.isfinite(scales).all(1) & (scales > 0).all(1) & np.isfinite(opacity) &
          np.isfinite(sh).all(axis=(1, 2)))
    if not ok.all():
        raise SceneFormatError(f"record {int(np.argmin(ok))}: non-finite or degenerate values")
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    return {"means": f32(means), "quats": f32(q), "scales": f32(scales),
            "opacity": f32(opacity), "sh": f32(sh)}


def load_ply(path) -> list:
    """scene_io.load_ply (scene_io.py:189-254): a list of Gaussian3D (API
    compatibility; render() also takes the arrays of load_ply_arrays)."""
    a = load_ply_arrays(path)
    return [Gaussian3D(mean=a["means"][i].astype(np.float64),
                       rotation=a["quats"][i].astype(np.float64),
                       scale=a["scales"][i].astype(np.float64),
                       opacity=float(a["opacity"][i]), sh=a["sh"][i].astype(np.float64))
            for i in range(len(a["opacity"]))]


def load_ply_scene(path, device=None):
    """Decode a checkpoint and upload it once: a device-resident
    GaussianScene for Renderer / render."""
    from .renderer import GaussianScene
    return GaussianScene.from_any(load_ply_arrays(path), device)


def _reorthonormalise(r: np.ndarray) -> np.ndarray:
    u = r[0] / np.linalg.norm(r[0])
    v = r[1] - (r[1] @ u) * u
    v /= np.linalg.norm(v)
    w = r[2] - (r[2] @ u) * u - (r[2] @ v) * v
    return np.stack([u, v, w / np.linalg.norm(w)])


def load_cameras(path, transpose: bool = False) -> list:
    """scene_io.load_cameras (scene_io.py:366-417): a JSON array of cameras
    (width, height, position, rotation world->view, fx, fy, optional cx, cy);
    ``transpose`` for stored view->world rotations; rotation drift up to 1e-3
    is re-orthonormalised, more is rejected."""
    try:
        items = json.loads(Path(path).read_text())
    except json.JSONDecodeError as e:
        raise SceneFormatError(f"camera file is not valid JSON: {e}") from e
    if not isinstance(items, list):
        raise SceneFormatError("camera file must hold a JSON array")
    out = []
    for i, c in enumerate(items):
        need = [k for k in ("width", "height", "position", "rotation", "fx", "fy") if k not in c]
        if need:
            raise SceneFormatError(f"camera entry {i} missing field {need[0]!r}")
        r = np.asarray(c["rotation"], dtype=np.float64)
        if r.shape != (3, 3):
            raise SceneFormatError(f"camera entry {i}: rotation must be 3x3")
        r = r.T if transpose else r
        err = float(np.abs(r @ r.T - np.eye(3)).max())
        if err > 1e-3:
            raise SceneFormatError(f"camera entry {i}: rotation drift {err:.3g} exceeds 1e-3 "
                                   f"(det {np.linalg.det(r):.6f})")
        if err > 1e-7:
            r = _reorthonormalise(r)
        out.append(Camera(rotation=r, position=np.asarray(c["position"], dtype=np.float64),
                          fx=c["fx"], fy=c["fy"], width=c["width"], height=c["height"],
                          cx=c.get("cx"), cy=c.get("cy")))
    return out
