"""View-consistency evaluation on the device (the
reference's metrics.py:80-255): analytic flow from rendered depth, bilinear
backward warping, the forward-backward occlusion test and the
warp-and-compare consistency score over a trajectory (the C5 popping
evaluation), as batched torch tensor ops on the frames the renderer already
holds on the GPU.  The squared-error score is supported; the FLIP score
(flip.py) is not and raises ConfigError.

Functions take numpy arrays or torch tensors and return torch tensors
(float64) on the input's device unless ``numpy=True``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .types import ConfigError, FrameOutput

BORDER_CROP = 20


def _t(x, device=None):
    if isinstance(x, torch.Tensor):
        return x.to(dtype=torch.float64, device=device or x.device)
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=device)


def analytic_flow(frame, cam_i, cam_j, device=None):
    """metrics.analytic_flow (metrics.py:218-255): each pixel of view i is
    pushed to the distance depth / (1 - T) along its ray and reprojected
    into view j.  Returns (flow[H,W,2] in pixels, valid[H,W]); pixels with
    T > 0.5, no positive distance or behind camera j are invalid, and flow is
    zeroed where it is not computable."""
    if frame.depth is None:
        raise ConfigError("analytic_flow needs a frame rendered with depth")
    depth = _t(frame.depth, device)
    dev = depth.device
    tn = _t(frame.transmittance, dev)
    h, w = depth.shape
    dist = depth / torch.clamp(1.0 - tn, min=1e-12)
    valid = (tn <= 0.5) & (dist > 0)
    ys, xs = torch.meshgrid(torch.arange(h, device=dev, dtype=torch.float64) + 0.5,
                            torch.arange(w, device=dev, dtype=torch.float64) + 0.5, indexing="ij")
    # rays_through_points (tile_culling.py:161-173): normalize(v @ R_i)
    Ri = _t(cam_i.rotation, dev)
    v = torch.stack([(xs - cam_i.cx) / cam_i.fx, (ys - cam_i.cy) / cam_i.fy,
                     torch.ones_like(xs)], dim=-1)
    d = v @ Ri
    d = d / torch.linalg.norm(d, dim=-1, keepdim=True)
    world = _t(cam_i.position, dev) + dist[..., None] * d
    rel = (world - _t(cam_j.position, dev)) @ _t(cam_j.rotation, dev).T
    z = rel[..., 2]
    front = z > 1e-9
    zs = torch.where(front, z, torch.ones_like(z))
    u = cam_j.fx * rel[..., 0] / zs + cam_j.cx
    vv = cam_j.fy * rel[..., 1] / zs + cam_j.cy
    flow = torch.stack([u - xs, vv - ys], dim=-1)
    flow = torch.where((front & (dist > 0))[..., None], flow, torch.zeros_like(flow))
    return flow, valid & front


def warp_frame(frame, flow, device=None):
    """metrics.warp_frame (metrics.py:80-106): out[p] = frame[p + flow[p]],
    bilinear with the sample clamped to the image (map_coordinates order 1,
    mode "nearest"); valid marks samples inside [0, W-1] x [0, H-1]."""
    f = _t(frame, device)
    fl = _t(flow, f.device)
    h, w = f.shape[:2]
    if tuple(fl.shape) != (h, w, 2):
        raise ConfigError(f"flow dims {tuple(fl.shape)} do not match frame {tuple(f.shape)}")
    ys, xs = torch.meshgrid(torch.arange(h, device=f.device, dtype=torch.float64),
                            torch.arange(w, device=f.device, dtype=torch.float64), indexing="ij")
    sx, sy = xs + fl[..., 0], ys + fl[..., 1]
    valid = (sx >= 0) & (sx <= w - 1) & (sy >= 0) & (sy <= h - 1)
    cx, cy = sx.clamp(0, w - 1), sy.clamp(0, h - 1)
    x0, y0 = cx.floor(), cy.floor()
    ax, ay = cx - x0, cy - y0
    x0i, y0i = x0.long(), y0.long()
    x1i, y1i = (x0i + 1).clamp(max=w - 1), (y0i + 1).clamp(max=h - 1)
    planar = f.dim() == 2
    g = f[..., None] if planar else f
    ax, ay = ax[..., None], ay[..., None]
    out = ((1 - ay) * ((1 - ax) * g[y0i, x0i] + ax * g[y0i, x1i]) +
           ay * ((1 - ax) * g[y1i, x0i] + ax * g[y1i, x1i]))
    return (out[..., 0] if planar else out), valid


def occlusion_mask(flow_fwd, flow_bwd, rel: float = 0.01, offset: float = 0.5, device=None):
    """metrics.occlusion_mask (metrics.py:109-125): usable where the round
    trip |f + b(p + f)|^2 <= rel (|f|^2 + |b|^2) + offset and in frame."""
    ff = _t(flow_fwd, device)
    bs, valid = warp_frame(flow_bwd, ff)
    lhs = ((ff + bs) ** 2).sum(-1)
    rhs = rel * ((ff ** 2).sum(-1) + (bs ** 2).sum(-1))
    return (lhs <= rhs + offset) & valid


def border_crop(height: int, width: int, crop: int = BORDER_CROP) -> int:
    """metrics.border_crop (metrics.py:128-133)."""
    side = min(height, width)
    return crop if side >= 64 else max(0, int(round(crop * side / 64)))


@dataclass
class ConsistencyReport:
    """metrics.ConsistencyReport: per-offset scores."""

    flip_t: dict
    mse_t: dict
    frames_used: int


def view_consistency(frames, flows_fwd: dict, flows_bwd: dict, offsets=(1, 7),
                     metric: str = "mse", crop: int | None = None,
                     device=None) -> ConsistencyReport:
    """metrics.view_consistency (metrics.py:145-215) with the squared-error
    score: frame i is compared with frame i+t warped onto it, over the
    cropped, flow-valid, occlusion-free pixels, after subtracting the
    per-pixel minimum over the sequence (static error cancels)."""
    if metric in ("flip", "both"):
        raise ConfigError("the FLIP score is not implemented on the B200 path; use metric='mse'")
    if metric != "mse":
        raise ConfigError(f"unknown metric {metric!r}")
    cols = [_t(f.color if isinstance(f, FrameOutput) else f, device) for f in frames]
    n = len(cols)
    offsets = (offsets,) if isinstance(offsets, int) else tuple(offsets)
    mse_t = {}
    for t in offsets:
        if t < 1:
            raise ConfigError(f"offset must be >= 1, got {t}")
        if n < t + 1:
            raise ConfigError(f"need at least {t + 1} frames for offset {t}, have {n}")
        h, w = cols[0].shape[:2]
        c = border_crop(h, w) if crop is None else crop
        maps, masks = [], []
        for i in range(n - t):
            j = i + t
            flow, fvalid = flows_fwd[(i, j)]
            flow = _t(flow, cols[0].device)
            fvalid = torch.as_tensor(fvalid, device=cols[0].device)
            warped, wvalid = warp_frame(cols[j], flow)
            bflow, bvalid = flows_bwd[(j, i)]
            usable = occlusion_mask(flow, _t(bflow, cols[0].device))
            bw, _ = warp_frame(torch.as_tensor(bvalid, device=cols[0].device).double(), flow)
            m = fvalid & wvalid & usable & (bw > 0.999)
            masks.append(m[c:h - c, c:w - c])
            maps.append(((cols[i] - warped) ** 2).mean(-1)[c:h - c, c:w - c])
        if not maps:
            continue
        st, ms = torch.stack(maps), torch.stack(masks)
        minmap = torch.where(ms, st, torch.full_like(st, float("inf"))).min(0).values
        vals = []
        for i in range(len(maps)):
            sel = ms[i] & torch.isfinite(minmap)
            if bool(sel.any()):
                vals.append(float((st[i][sel] - minmap[sel]).mean()))
        mse_t[t] = float(np.mean(vals)) if vals else 0.0
    return ConsistencyReport(flip_t={}, mse_t=mse_t, frames_used=n)
