"""View-consistency evaluation on the device (the
reference's metrics.py:80-255): analytic flow from rendered depth, bilinear
backward warping, the forward-backward occlusion test and the
warp-and-compare consistency score over a trajectory (the C5 popping
evaluation), as batched torch tensor ops on the frames the renderer already
holds on the GPU, with the FLIP perceptual difference (flip.py) restated in
torch (``flip_error_map``) and the squared-error score.

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


# ---------------------------------------------------------------------------
# FLIP perceptual difference (flip.py): the colour pipeline (CSF-filtered
# opponent channels, Hunt-adjusted L*a*b*, HyAB distance redistributed around
# the green/blue maximum) and the feature pipeline (edge / point detector
# magnitudes of the achromatic channel), combined as dc ** (1 - df).

_M_SRGB2XYZ = torch.tensor([[0.41238656, 0.35759149, 0.18045049],
                            [0.21263682, 0.71518298, 0.07218020],
                            [0.01933062, 0.11919716, 0.95037259]], dtype=torch.float64)


def _white(dev):
    return (_M_SRGB2XYZ.to(dev) @ torch.ones(3, dtype=torch.float64, device=dev))


def _lin(img):
    x = img.clamp(0.0, 1.0)
    return torch.where(x <= 0.04045, x / 12.92, ((x + 0.055) / 1.055) ** 2.4)


def _xyz(rgb):
    return rgb @ _M_SRGB2XYZ.to(rgb.device).T


def _ycxcz(xyz):
    n = xyz / _white(xyz.device)
    return torch.stack([116.0 * n[..., 1] - 16.0, 500.0 * (n[..., 0] - n[..., 1]),
                        200.0 * (n[..., 1] - n[..., 2])], dim=-1)


def _ycxcz_to_rgb(v):
    yn = (v[..., 0] + 16.0) / 116.0
    xyz = torch.stack([v[..., 1] / 500.0 + yn, yn, yn - v[..., 2] / 200.0], dim=-1)
    xyz = xyz * _white(v.device)
    return xyz @ torch.linalg.inv(_M_SRGB2XYZ.to(v.device)).T


def _lab_hunt(xyz):
    n = xyz / _white(xyz.device)
    d = 6.0 / 29.0
    f = torch.where(n > d ** 3, torch.sign(n) * n.abs() ** (1.0 / 3.0), n / (3 * d * d) + 4.0 / 29.0)
    L = 116.0 * f[..., 1] - 16.0
    s = L / 100.0
    return torch.stack([L, 500.0 * (f[..., 0] - f[..., 1]) * s,
                        200.0 * (f[..., 1] - f[..., 2]) * s], dim=-1)


def _hyab(a, b):
    d = a - b
    return d[..., 0].abs() + torch.sqrt(d[..., 1] ** 2 + d[..., 2] ** 2)


def _csf(a1, b1, a2, b2, ppd, dev):
    r = int(np.ceil(3 * np.sqrt(0.04 / (2 * np.pi ** 2)) * ppd))
    t = torch.arange(-r, r + 1, dtype=torch.float64, device=dev) / ppd
    zz = t[None, :] ** 2 + t[:, None] ** 2
    g = (a1 * np.sqrt(np.pi / b1) * torch.exp(-np.pi ** 2 * zz / b1) +
         a2 * np.sqrt(np.pi / b2) * torch.exp(-np.pi ** 2 * zz / b2))
    return g / g.sum()


def _detectors(ppd, dev):
    sd = 0.5 * 0.082 * ppd
    r = int(np.ceil(3 * sd))
    t = torch.arange(-r, r + 1, dtype=torch.float64, device=dev)
    x, y = t[None, :].expand(2 * r + 1, -1), t[:, None].expand(-1, 2 * r + 1)
    g = torch.exp(-(x * x + y * y) / (2 * sd * sd))

    def unit(k):  # negative lobe sums to -1, positive to +1
        neg, pos = -k[k < 0].sum(), k[k > 0].sum()
        return torch.where(k < 0, k / neg, k / pos)

    return unit(-x * g), unit((x * x / (sd * sd) - 1) * g)


def _conv(img, k):
    """scipy.ndimage.convolve(img, k, mode="reflect") for a 2D plane: true
    convolution, the border mirrored including the edge sample."""
    ry, rx = k.shape[0] // 2, k.shape[1] // 2
    h, w = img.shape

    def sym(n, r):
        i = torch.arange(-r, n + r, device=img.device)
        m = 2 * n
        i = torch.remainder(i, m)
        return torch.where(i >= n, m - 1 - i, i)

    p = img[sym(h, ry)][:, sym(w, rx)]
    kf = torch.flip(k, dims=(0, 1))
    return torch.nn.functional.conv2d(p[None, None], kf[None, None])[0, 0]


def flip_error_map(a, b, ppd: float = 67.0, device=None):
    """flip.flip_error_map (flip.py:105-156): per-pixel perceptual difference
    in [0, 1] of two RGB images in [0, 1], viewed at ``ppd`` pixels/degree."""
    A, B = _t(a, device), _t(b, device)
    if A.shape != B.shape or A.dim() != 3 or A.shape[2] != 3:
        raise ValueError(f"need matching HxWx3 images, got {tuple(A.shape)} and {tuple(B.shape)}")
    dev = A.device
    ks = (_csf(1.0, 0.0047, 0.0, 1e-5, ppd, dev), _csf(1.0, 0.0053, 0.0, 1e-5, ppd, dev),
          _csf(34.1, 0.04, 13.5, 0.025, ppd, dev))

    def colour(img):
        v = _ycxcz(_xyz(_lin(img)))
        f = torch.stack([_conv(v[..., c], ks[c]) for c in range(3)], dim=-1)
        return _lab_hunt(_xyz(_ycxcz_to_rgb(f).clamp(0.0, 1.0)))

    qc, qf, pc, pt = 0.7, 0.5, 0.4, 0.95
    d = _hyab(colour(A), colour(B))
    g = _lab_hunt(_xyz(torch.tensor([[[0.0, 1.0, 0.0]]], dtype=torch.float64, device=dev)))
    bl = _lab_hunt(_xyz(torch.tensor([[[0.0, 0.0, 1.0]]], dtype=torch.float64, device=dev)))
    cmax = float(_hyab(g, bl).reshape(()) ** qc)
    dc = d ** qc
    dc = torch.where(dc < pc * cmax, (pt / (pc * cmax)) * dc,
                     pt + ((dc - pc * cmax) / (cmax - pc * cmax)) * (1.0 - pt))
    ke, kp = _detectors(ppd, dev)

    def ach(img):
        return (_ycxcz(_xyz(_lin(img)))[..., 0] + 16.0) / 116.0

    def mag(y, k):
        return torch.sqrt(_conv(y, k) ** 2 + _conv(y, k.T) ** 2)

    ya, yb = ach(A), ach(B)
    df = (torch.maximum((mag(ya, ke) - mag(yb, ke)).abs(), (mag(ya, kp) - mag(yb, kp)).abs())
          / np.sqrt(2.0)) ** qf
    return (dc ** (1.0 - df)).clamp(0.0, 1.0)


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
                     metric: str = "both", crop: int | None = None,
                     device=None) -> ConsistencyReport:
    """metrics.view_consistency (metrics.py:145-215), FLIP and / or
    squared-error scores: frame i is compared with frame i+t warped onto it, over the
    cropped, flow-valid, occlusion-free pixels, after subtracting the
    per-pixel minimum over the sequence (static error cancels)."""
    if metric not in ("flip", "mse", "both"):
        raise ConfigError(f"unknown metric {metric!r}")
    cols = [_t(f.color if isinstance(f, FrameOutput) else f, device) for f in frames]
    n = len(cols)
    offsets = (offsets,) if isinstance(offsets, int) else tuple(offsets)
    mse_t, flip_t = {}, {}
    for t in offsets:
        if t < 1:
            raise ConfigError(f"offset must be >= 1, got {t}")
        if n < t + 1:
            raise ConfigError(f"need at least {t + 1} frames for offset {t}, have {n}")
        h, w = cols[0].shape[:2]
        c = border_crop(h, w) if crop is None else crop
        maps, fmaps, masks = [], [], []
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
            if metric in ("flip", "both"):
                fmaps.append(flip_error_map(cols[i], warped)[c:h - c, c:w - c])
            if metric in ("mse", "both"):
                maps.append(((cols[i] - warped) ** 2).mean(-1)[c:h - c, c:w - c])
        for mp, out in ((fmaps, flip_t), (maps, mse_t)):
            if not mp:
                continue
            st, ms = torch.stack(mp), torch.stack(masks)
            minmap = torch.where(ms, st, torch.full_like(st, float("inf"))).min(0).values
            vals = []
            for i in range(len(mp)):
                sel = ms[i] & torch.isfinite(minmap)
                if bool(sel.any()):
                    vals.append(float((st[i][sel] - minmap[sel]).mean()))
            out[t] = float(np.mean(vals)) if vals else 0.0
    return ConsistencyReport(flip_t=flip_t, mse_t=mse_t, frames_used=n)
