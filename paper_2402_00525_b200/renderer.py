"""Drop-in ``render`` for the reference's Hierarchical forward path, on B200.

Mirrors ``splatsort.render(scene, cam, mode, cfg) -> FrameOutput``
(rasterizer.py:595-698), ``render_depth`` (:701-715) and ``render_trajectory``
(:758-772).  The heavy lifting is one C-ABI call per view (include/stp.h ->
libstp_b200.so, hand-written sm_100a kernels K1..K6); this module only
stages tensors, owns the device workspace, and converts outputs.

There is no CPU fallback: without a CUDA device or the built library every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .types import (Camera, ConfigError, DataError, FrameOutput, FullPerPixel, Hierarchical,
                    PixelRecords, RenderConfig, _is_hier, mode_name, validate_mode)

_SH_OK = (1, 4, 9, 16)


def _require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2402_00525_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise RuntimeError("device must be a CUDA device")
    return dev


class GaussianScene:
    """Device-resident Gaussians in the drop-in tensor layout (float32):
    means[N,3], quats[N,4] (w,x,y,z), scales[N,3], opacity[N], sh[N,K,3]."""

    def __init__(self, means, quats, scales, opacity, sh, device=None):
        dev = _require_cuda(device)

        def t(a, shape_tail):
            x = torch.as_tensor(a) if not isinstance(a, torch.Tensor) else a
            x = x.to(device=dev, dtype=torch.float32).contiguous()
            return x.reshape(-1, *shape_tail) if shape_tail else x.reshape(-1)

        self.means = t(means, (3,))
        self.quats = t(quats, (4,))
        self.scales = t(scales, (3,))
        self.opacity = t(opacity, ())
        n = self.means.shape[0]
        sh_t = torch.as_tensor(sh) if not isinstance(sh, torch.Tensor) else sh
        sh_t = sh_t.to(device=dev, dtype=torch.float32)
        sh_t = sh_t.reshape(n, -1, 3) if n else sh_t.reshape(0, 16, 3)[:, :16]
        k = sh_t.shape[1] if n else 16
        if k not in _SH_OK:
            raise DataError(f"sh must hold 1, 4, 9 or 16 coefficients per channel, got {k}")
        self.sh = sh_t.contiguous()
        for name, x in (("quats", self.quats), ("scales", self.scales),
                        ("opacity", self.opacity)):
            if x.shape[0] != n:
                raise DataError(f"{name} has {x.shape[0]} rows, means has {n}")
        self.device = dev

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    @property
    def sh_coeffs(self) -> int:
        return int(self.sh.shape[1]) if self.n else 16

    @classmethod
    def from_any(cls, scene, device=None) -> "GaussianScene":
        if isinstance(scene, GaussianScene):
            return scene
        if isinstance(scene, dict):
            return cls(scene["means"], scene["quats"], scene["scales"], scene["opacity"],
                       scene["sh"], device)
        gs = list(scene)
        if not gs:
            z = np.zeros
            return cls(z((0, 3)), z((0, 4)), z((0, 3)), z(0), z((0, 16, 3)), device)
        return cls(np.stack([np.asarray(g.mean, dtype=np.float64) for g in gs]),
                   np.stack([np.asarray(g.rotation, dtype=np.float64) for g in gs]),
                   np.stack([np.asarray(g.scale, dtype=np.float64) for g in gs]),
                   np.array([float(g.opacity) for g in gs]),
                   np.stack([np.asarray(g.sh, dtype=np.float64).reshape(-1, 3) for g in gs]),
                   device)

    def struct(self) -> _lib.StpScene:
        s = _lib.StpScene()
        s.means = self.means.data_ptr()
        s.quats = self.quats.data_ptr()
        s.scales = self.scales.data_ptr()
        s.opacity = self.opacity.data_ptr()
        s.sh = self.sh.data_ptr()
        s.n = self.n
        s.sh_coeffs = self.sh_coeffs
        return s


class BatchScene:
    """Device copy (float64) of an already-projected SplatBatch
    (gaussian_math.py:260-307; duck-typed: the reference's own SplatBatch or
    this package's).  Rendered through stp_render_batch, which skips the
    projection like rasterizer.py:616-618."""

    FIELDS = ("mean2d", "conic", "color", "opacity", "radius", "inv_cov3", "inv_cov_center")

    def __init__(self, batch, device=None):
        dev = _require_cuda(device)
        n = len(batch.opacity)
        shapes = {"mean2d": (n, 2), "conic": (n, 3), "color": (n, 3), "opacity": (n,),
                  "radius": (n,), "inv_cov3": (n, 6), "inv_cov_center": (n, 3)}
        self.t = {}
        for k in self.FIELDS:
            a = torch.as_tensor(np.ascontiguousarray(getattr(batch, k), dtype=np.float64))
            if tuple(a.shape) != shapes[k]:
                raise DataError(f"SplatBatch.{k} has shape {tuple(a.shape)}, expected {shapes[k]}")
            self.t[k] = a.to(dev).contiguous()
        # GlobalZ inputs (view z keys, distance depth), when the batch has them
        for k in ("global_depth", "center_dist"):
            v = getattr(batch, k, None)
            if v is not None:
                a = torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64))
                if tuple(a.shape) != (n,):
                    raise DataError(f"SplatBatch.{k} has shape {tuple(a.shape)}, expected {(n,)}")
                self.t[k] = a.to(dev).contiguous()
        self.source_index = np.asarray(batch.source_index, dtype=np.int64).copy()
        self.device = dev

    @property
    def n(self) -> int:
        return int(self.t["opacity"].shape[0])

    def struct(self) -> _lib.StpSplatBatch:
        b = _lib.StpSplatBatch()
        for k in self.FIELDS:
            setattr(b, k, self.t[k].data_ptr())
        b.n = self.n
        for k in ("global_depth", "center_dist"):
            setattr(b, k, self.t[k].data_ptr() if k in self.t else None)
        return b


def _is_globalz(mode) -> bool:
    return type(mode).__name__ == "GlobalZ"


WINDOW_MAX = 512   # stp.h STP_WINDOW_MAX: register window <= 16, shared-memory heap above


def _check_supported(mode) -> None:
    """All four sort modes run on the B200 path: Hierarchical (the paper's
    pipeline), GlobalZ (the 3DGS order), FullPerPixel (the exact per-pixel
    order) and Window(size) with 1 <= size <= WINDOW_MAX."""
    if type(mode).__name__ == "Window" and not 1 <= int(mode.size) <= WINDOW_MAX:
        raise ConfigError(f"the B200 Window mode keeps at most {WINDOW_MAX} entries per pixel, "
                          f"got {mode_name(mode)}")


def _is_batch(scene) -> bool:
    return isinstance(scene, BatchScene) or (hasattr(scene, "mean2d") and
                                             hasattr(scene, "inv_cov3"))


def make_camera(cam) -> _lib.StpCamera:
    c = _lib.StpCamera()
    R = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
    for i in range(9):
        c.R[i] = float(R[i])
    p = np.asarray(cam.position, dtype=np.float64).reshape(3)
    for i in range(3):
        c.pos[i] = float(p[i])
    c.fx, c.fy = float(cam.fx), float(cam.fy)
    c.cx = float(cam.cx) if cam.cx is not None else cam.width / 2.0
    c.cy = float(cam.cy) if cam.cy is not None else cam.height / 2.0
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def make_config(cfg: RenderConfig, mode, record_cap: int = 0, timings: bool = False,
                tiles=None):
    c = _lib.StpConfig()
    c.eps = float(cfg.opacity_eps)
    c.termination = float(cfg.termination)
    c.alpha_cap = float(cfg.alpha_cap)
    bg = np.asarray(cfg.background, dtype=np.float64).reshape(3)
    for i in range(3):
        c.bg[i] = float(bg[i])
    c.near_plane = float(cfg.near)
    c.guard = float(cfg.guard_band)
    c.dilation = float(cfg.dilation)
    c.inv_scale_clamp = float(cfg.inv_scale_clamp)
    c.tile_size = int(cfg.tile_size)
    q = mode if _is_hier(mode) else Hierarchical()  # other modes: queue fields unused
    c.q_tail, c.q_mid, c.q_head = int(q.queue_tail), int(q.queue_mid), int(q.queue_head)
    c.b_load, c.b_mid, c.b_head = int(q.batch_load), int(q.batch_mid), int(q.batch_head)
    c.mid_depth_at_center = int(bool(q.mid_depth_at_center))
    name = type(mode).__name__
    c.sort_mode = {"GlobalZ": _lib.STP_MODE_GLOBALZ, "FullPerPixel": _lib.STP_MODE_FULL,
                   "Window": _lib.STP_MODE_WINDOW}.get(name, _lib.STP_MODE_HIERARCHICAL)
    if name == "Window":
        c.q_head = int(mode.size)  # the window size (stp.h STP_MODE_WINDOW)
    if tiles is not None:          # K6 tile band [t0, t1) (multi-GPU view split)
        c.tile_begin, c.tile_end = int(tiles[0]), int(tiles[1])
    c.with_depth = int(bool(cfg.with_depth))
    c.exact_culling = int(bool(cfg.exact_culling(mode)))
    c.record_cap = int(record_cap)
    c.flags = _lib.STP_FLAG_TIMINGS if timings else 0
    return c


def _raise(code: int, what: str):
    msg = f"{what}: {_lib.error_string(code)}"
    if code == _lib.STP_ERR_CONFIG:
        raise ConfigError(msg)
    raise DataError(msg)


class Workspace:
    """Caller-owned device workspace (one per device/stream), grown on demand."""

    def __init__(self, device):
        self.device = device
        self.buf = torch.empty(0, dtype=torch.uint8, device=device)

    def ensure(self, n: int, width: int, height: int, entries: int) -> None:
        need = int(_lib.load().stp_workspace_bytes(n, width, height, int(entries)))
        if self.buf.numel() < need:
            self.buf = torch.zeros(need, dtype=torch.uint8, device=self.device)  # zeroed once: the sort look-back words are epoch-tagged, never cleared per frame

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    @property
    def nbytes(self) -> int:
        return self.buf.numel()

    def layout(self, n, width, height) -> _lib.StpLayout:
        L = _lib.StpLayout()
        rc = _lib.load().stp_workspace_layout(n, width, height, self.nbytes, ctypes.byref(L))
        if rc != _lib.STP_OK:
            _raise(rc, "workspace layout")
        return L


_WORKSPACES: dict = {}


def workspace_for(device) -> Workspace:
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    ws = _WORKSPACES.get(key)
    if ws is None:
        ws = _WORKSPACES[key] = Workspace(device)
    return ws


class Renderer:
    """Renders views of one device-resident scene; the building block of
    ``render``, the multi-view driver and the benchmark.

    ``render_into`` is asynchronous (no host sync) unless stats are requested;
    an asynchronous frame's entry overflow is reported by the device status
    word (``check_status``).  The default mode of this class is Hierarchical
    (the B200 hot path); the drop-in ``render`` defaults to FullPerPixel like
    the reference.
    """

    def __init__(self, scene, mode=None, cfg: RenderConfig | None = None, device=None,
                 entry_capacity: int | None = None):
        if _is_batch(scene):
            self.scene = scene if isinstance(scene, BatchScene) else BatchScene(scene, device)
        else:
            self.scene = GaussianScene.from_any(scene, device)
        self.batch = isinstance(self.scene, BatchScene)
        self.device = self.scene.device
        self.mode = mode if mode is not None else Hierarchical()
        validate_mode(self.mode)
        _check_supported(self.mode)
        if _is_globalz(self.mode) and self.batch and not {"global_depth", "center_dist"} <= \
                set(self.scene.t):
            raise DataError("GlobalZ needs SplatBatch.global_depth and center_dist")
        self.cfg = cfg if cfg is not None else RenderConfig()
        self.lib = _lib.load()
        self.ws = Workspace(self.device)
        self.entry_capacity = entry_capacity
        # StpOutputs.status of the asynchronous path: (code, entries), written by K5
        self.status = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.c_scene = self.scene.struct()
        rc = self.lib.stp_validate_config(ctypes.byref(make_config(self.cfg, self.mode)))
        if rc != _lib.STP_OK:
            _raise(rc, "configuration")

    def alloc_outputs(self, width, height, record_cap: int = 0, with_state: bool = False,
                      sort_error: bool = False, f64: bool = False):
        """Device output buffers for render_into.  ``f64``: also the float64
        outputs (StpOutputs.color64 ...: colour / depth accumulated and the
        background composited in float64, records' t and alpha in float64 --
        the reference's FrameOutput precision)."""
        d = self.device
        o = {"color": torch.empty((height, width, 3), dtype=torch.float32, device=d),
             "transmittance": torch.empty((height, width), dtype=torch.float32, device=d)}
        if self.cfg.with_depth:
            o["depth"] = torch.empty((height, width), dtype=torch.float32, device=d)
        if record_cap > 0:
            o["rec_count"] = torch.empty((height, width), dtype=torch.int32, device=d)
            o["rec_splat"] = torch.empty((height, width, record_cap), dtype=torch.int32, device=d)
            o["rec_t"] = torch.empty((height, width, record_cap), dtype=torch.float32, device=d)
            o["rec_alpha"] = torch.empty((height, width, record_cap), dtype=torch.float32, device=d)
        if with_state:
            o["state"] = torch.empty(max(1, self.scene.n), dtype=torch.uint8, device=d)
        if sort_error:
            o["sort_error"] = torch.empty((height, width), dtype=torch.float32, device=d)
        if f64:
            f = torch.float64
            o["color64"] = torch.empty((height, width, 3), dtype=f, device=d)
            if not self.batch:
                o["splat_color64"] = torch.empty((max(1, self.scene.n), 3), dtype=f, device=d)
            o["transmittance64"] = torch.empty((height, width), dtype=f, device=d)
            if self.cfg.with_depth:
                o["depth64"] = torch.empty((height, width), dtype=f, device=d)
            if record_cap > 0:
                o["rec_t64"] = torch.empty((height, width, record_cap), dtype=f, device=d)
                o["rec_alpha64"] = torch.empty((height, width, record_cap), dtype=f, device=d)
        return o

    @staticmethod
    def outputs_struct(o: dict) -> _lib.StpOutputs:
        s = _lib.StpOutputs()
        for k in ("color", "transmittance", "depth", "rec_count", "rec_splat", "rec_t",
                  "rec_alpha", "state", "sort_error", "status", "color64", "transmittance64",
                  "depth64", "rec_t64", "rec_alpha64", "splat_color64"):
            if k in o:
                setattr(s, k, o[k].data_ptr())
        return s

    def _ensure(self, cam):
        guess = self.entry_capacity or max(1 << 16, 8 * self.scene.n)
        self._last_w, self._last_h = int(cam.width), int(cam.height)
        self.ws.ensure(self.scene.n, cam.width, cam.height, guess)

    def render_into(self, cam, outs: dict, stats: bool = False, timings: bool = False,
                    record_cap: int = 0, stream=None, tiles=None):
        """One view into preallocated device outputs.  Returns StpStats when
        ``stats`` (synchronising; an entry overflow grows the workspace and
        re-renders), else None (asynchronous: the frame's status word lands in
        ``self.status`` -- see ``check_status``).  ``tiles`` = (t0, t1)
        renders only that band of row-major tile ids (the pixels of the other
        tiles are left untouched)."""
        c_cam = make_camera(cam)
        self._ensure(cam)
        if not record_cap and "rec_splat" in outs:
            record_cap = int(outs["rec_splat"].shape[2])   # the buffers' capacity
        if record_cap and "rec_splat" not in outs:
            raise DataError("record_cap > 0 needs record buffers (alloc_outputs(record_cap=...))")
        c_cfg = make_config(self.cfg, self.mode, record_cap, timings, tiles)
        c_out = self.outputs_struct(outs)
        if "status" not in outs:
            c_out.status = self.status.data_ptr()
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        st = _lib.StpStats() if stats else None
        for attempt in range(3):
            fn = self.lib.stp_render_batch if self.batch else self.lib.stp_render
            rc = fn(ctypes.byref(self.c_scene), ctypes.byref(c_cam),
                    ctypes.byref(c_cfg), ctypes.c_void_p(self.ws.ptr),
                    self.ws.nbytes, ctypes.byref(c_out),
                    ctypes.byref(st) if st is not None else None,
                    ctypes.c_void_p(s))
            if rc == _lib.STP_ERR_WORKSPACE_TOO_SMALL and st is not None:
                need = int(st.bin_entries * 1.25) + 4096
                self.entry_capacity = need
                self.ws.ensure(self.scene.n, cam.width, cam.height, need)
                continue
            if rc != _lib.STP_OK:
                _raise(rc, "stp_render")
            return st
        raise DataError("stp_render: workspace retry failed")

    def render_views(self, cams, outs_list, stream=None, retry: bool = True):
        """``render_trajectory``'s loop of independent views (rasterizer.py:
        758-772) as ONE stp_render_views call on one stream (one workspace,
        outputs per view, no host sync inside).  Each view's status word is
        written on the device; with ``retry`` the call synchronises once at
        the end and re-renders the views that overflowed the workspace (grown
        to the largest entry count).  Returns the [V, 2] status tensor."""
        V = len(cams)
        if V != len(outs_list):
            raise DataError("render_views: one output dict per camera")
        if self.batch:
            raise DataError("render_views takes a Gaussian scene, not a SplatBatch")
        status = torch.zeros((max(V, 1), 2), dtype=torch.int64, device=self.device)
        c_cams = (_lib.StpCamera * max(V, 1))()
        c_outs = (_lib.StpOutputs * max(V, 1))()
        for v, (cam, o) in enumerate(zip(cams, outs_list)):
            c_cams[v] = make_camera(cam)
            c_outs[v] = self.outputs_struct(o)
            c_outs[v].status = status[v].data_ptr()
        if V:
            self._ensure(cams[0])
            if any((c.width, c.height) != (cams[0].width, cams[0].height) for c in cams):
                w = max(c.width for c in cams)
                h = max(c.height for c in cams)
                self._last_w, self._last_h = w, h
                self.ws.ensure(self.scene.n, w, h, self.entry_capacity or 8 * self.scene.n)
        c_cfg = make_config(self.cfg, self.mode)
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        rc = self.lib.stp_render_views(ctypes.byref(self.c_scene), c_cams, V, ctypes.byref(c_cfg),
                                       ctypes.c_void_p(self.ws.ptr), self.ws.nbytes, c_outs,
                                       ctypes.c_void_p(s))
        if rc != _lib.STP_OK:
            _raise(rc, "stp_render_views")
        if retry and V:
            st = status[:V].cpu()
            bad = [v for v in range(V) if int(st[v, 0]) != _lib.STP_OK]
            if bad:
                if any(int(st[v, 0]) != _lib.STP_ERR_WORKSPACE_TOO_SMALL for v in bad):
                    _raise(int(st[bad[0], 0]), "stp_render_views (device status)")
                need = int(max(int(st[v, 1]) for v in bad) * 1.25) + 4096
                self.entry_capacity = max(self.entry_capacity or 0, need)
                for v in bad:
                    self.ws.ensure(self.scene.n, cams[v].width, cams[v].height,
                                   self.entry_capacity)
                    self.render_into(cams[v], outs_list[v], stats=True)
                    status[v, 0] = _lib.STP_OK
        return status[:V]

    def check_status(self, status=None, grow: bool = True) -> bool:
        """Read the status word of the last asynchronous frame (synchronises
        the stream).  True when the frame is complete; on an entry overflow
        the workspace is grown to the frame's entry count (``grow``) and False
        is returned -- the caller re-renders that view.  A scheduler fault
        raises DataError."""
        st = self.status if status is None else status
        code, entries = (int(x) for x in st.tolist())
        if code == _lib.STP_OK:
            return True
        if code == _lib.STP_ERR_WORKSPACE_TOO_SMALL:
            if grow:
                need = int(entries * 1.25) + 4096
                self.entry_capacity = max(self.entry_capacity or 0, need)
                self.ws.ensure(self.scene.n, self._last_w, self._last_h, self.entry_capacity)
            return False
        _raise(code, "stp_render (device status)")

    def frame(self, cam, device_output: bool = False, sort_error: bool = False) -> FrameOutput:
        """One frame.  ``sort_error``: also the per-pixel sort error delta
        (metrics.py:46-73), accumulated in the blend (FrameOutput.sort_error,
        stats["sort_error"] = delta_max / delta_avg)."""
        cfg = self.cfg
        t0 = time.perf_counter()
        rec_cap = 64 if cfg.capture_records else 0
        while True:
            # the float64 FrameOutput of the reference (rasterizer.py:246-255):
            # float64 colour / depth sums and records; device tensors stay fp32
            outs = self.alloc_outputs(cam.width, cam.height, rec_cap, with_state=True,
                                      sort_error=sort_error, f64=not device_output)
            st = self.render_into(cam, outs, stats=True, timings=True, record_cap=rec_cap)
            if rec_cap and int(outs["rec_count"].max().item()) > rec_cap:
                rec_cap = int(outs["rec_count"].max().item())
                continue
            break
        if self.batch:
            kept = torch.as_tensor(self.scene.source_index, device=self.device)
        else:
            state = outs["state"][: self.scene.n]
            kept = torch.nonzero(state == 0).flatten()
        timings = {"project": st.ms_project / 1e3, "duplicate": st.ms_duplicate / 1e3,
                   "sort": st.ms_sort / 1e3, "blend": st.ms_blend / 1e3}
        stats = {
            "mode": mode_name(self.mode),
            # a SplatBatch input reports only "kept" (rasterizer.py:616-618)
            "projection": ({"kept": int(st.kept)} if self.batch else
                           {"input": int(st.input), "behind": int(st.behind),
                            "guard": int(st.guard), "degenerate": int(st.degenerate),
                            "kept": int(st.kept)}),
            "bin_entries": int(st.bin_entries),
            "tiles": int(st.tiles),
            "timings": timings,
            "nonfinite_pixels": [],
            "tie_runs": int(st.tie_runs),
        }
        if st.nonfinite_pixels:
            bad = ~(torch.isfinite(outs["color"]).all(dim=2) & torch.isfinite(outs["transmittance"]))
            ys, xs = (t.cpu().numpy() for t in torch.nonzero(bad, as_tuple=True))
            stats["nonfinite_pixels"] = [(int(x), int(y)) for y, x in zip(ys, xs)]
        if sort_error:
            se = outs["sort_error"]
            stats["sort_error"] = {"delta_max": float(se.max().item()) if se.numel() else 0.0,
                                   "delta_avg": float(se.double().mean().item())
                                   if se.numel() else 0.0}
        if device_output:
            out = FrameOutput(color=outs["color"], transmittance=outs["transmittance"],
                              depth=outs.get("depth"), source_index=kept, stats=stats,
                              sort_error=outs.get("sort_error"))
            if rec_cap:
                out.records = {k: outs[k] for k in ("rec_count", "rec_splat", "rec_t",
                                                    "rec_alpha")}
            timings["total"] = time.perf_counter() - t0
            return out
        color = outs["color64"].cpu().numpy()
        tn = outs["transmittance64"].cpu().numpy()
        depth = outs["depth64"].cpu().numpy() if cfg.with_depth else None
        src = self.scene.source_index if self.batch else kept.cpu().numpy().astype(np.int64)
        records = None
        if rec_cap:
            records = self._records(outs, None if self.batch else src, cam)
        timings["total"] = time.perf_counter() - t0
        se = outs["sort_error"].double().cpu().numpy() if sort_error else None
        return FrameOutput(color=color, transmittance=tn, depth=depth, records=records,
                           source_index=src, stats=stats, sort_error=se)

    def backward(self, cam, upstream):
        """Gradients of the loss w.r.t. the projected splat attributes
        (gradients.py:103-162) for dL/d(colour) ``upstream`` [H,W,3]: the frame
        is re-rendered and K6 replayed (stp_backward); returns the per-splat
        SplatGradients in batch (kept-splat) order, float64 numpy."""
        from .gradients import SplatGradients
        H, W = int(cam.height), int(cam.width)
        up = torch.as_tensor(upstream, dtype=torch.float64).to(self.device).contiguous()
        if tuple(up.shape) != (H, W, 3):
            raise DataError(f"upstream gradient dims {tuple(up.shape)} do not match the frame")
        n = self.scene.n
        d = self.device
        pix = torch.empty((H, W, 4), dtype=torch.float64, device=d)
        gt = {k: torch.empty((max(n, 1), c), dtype=torch.float64, device=d)
              for k, c in (("d_color", 3), ("d_opacity", 1), ("d_mean2d", 2), ("d_conic", 3))}
        g = _lib.StpGrads()
        g.upstream, g.pix_state = up.data_ptr(), pix.data_ptr()
        for k, t in gt.items():
            setattr(g, k, t.data_ptr())
        outs = self.alloc_outputs(W, H, with_state=True)
        c_cam = make_camera(cam)
        self._ensure(cam)
        c_cfg = make_config(self.cfg, self.mode)
        c_out = self.outputs_struct(outs)
        s = torch.cuda.current_stream(d).cuda_stream
        st = _lib.StpStats()
        fn = self.lib.stp_backward_batch if self.batch else self.lib.stp_backward
        for _ in range(3):
            rc = fn(ctypes.byref(self.c_scene), ctypes.byref(c_cam), ctypes.byref(c_cfg),
                    ctypes.c_void_p(self.ws.ptr), self.ws.nbytes, ctypes.byref(c_out),
                    ctypes.byref(g), ctypes.byref(st), ctypes.c_void_p(s))
            if rc == _lib.STP_ERR_WORKSPACE_TOO_SMALL:
                need = int(st.bin_entries * 1.25) + 4096
                self.entry_capacity = need
                self.ws.ensure(self.scene.n, cam.width, cam.height, need)
                continue
            if rc != _lib.STP_OK:
                _raise(rc, "stp_backward")
            break
        else:
            raise DataError("stp_backward: workspace retry failed")
        if st.nonfinite_pixels:
            raise DataError("non-finite gradient or pixel in the backward pass")
        if self.batch:
            kept = torch.arange(n, device=d)
        else:
            kept = torch.nonzero(outs["state"][:n] == 0).flatten()
        f = lambda k: gt[k][kept].cpu().numpy()  # noqa: E731
        d_bg = (up * pix[..., 3:4]).sum(dim=(0, 1)).cpu().numpy()
        return SplatGradients(d_color=f("d_color"), d_opacity=f("d_opacity")[:, 0],
                              d_mean2d=f("d_mean2d"), d_conic=f("d_conic"), d_background=d_bg)

    def debug_bins(self, cam):
        """Sorted (tile_id, gaussian_id, fp32 key bits) of the last frame rendered
        with this renderer's workspace (parity dumps of K3-K5)."""
        torch.cuda.current_stream(self.device).synchronize()
        L = self.ws.layout(self.scene.n, cam.width, cam.height)
        st = _lib.StpStats()
        rc = self.lib.stp_read_stats(ctypes.c_void_p(self.ws.ptr), self.ws.nbytes, self.scene.n,
                                     cam.width, cam.height, ctypes.byref(st),
                                     ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        if rc != _lib.STP_OK:
            _raise(rc, "stp_read_stats")
        E = int(st.bin_entries)
        ko = L.keys1 if L.final_buffer else L.keys0
        vo = L.vals
        keys = self.ws.buf[ko: ko + 8 * E].view(torch.int64).cpu().numpy().view(np.uint64)
        vals = self.ws.buf[vo: vo + 4 * E].view(torch.int32).cpu().numpy()
        db, ib = np.uint64(L.depth_bits), np.uint64(L.id_bits)
        key = keys >> ib
        return (key >> db).astype(np.int64), vals.astype(np.int64), \
            ((key & ((np.uint64(1) << db) - np.uint64(1))) << (np.uint64(32) - db)).astype(np.uint32)

    @staticmethod
    def _records(outs, src, cam):
        cnt = outs["rec_count"].cpu().numpy()
        spl = outs["rec_splat"].cpu().numpy()
        tt = outs["rec_t64" if "rec_t64" in outs else "rec_t"].double().cpu().numpy()
        aa = outs["rec_alpha64" if "rec_alpha64" in outs else "rec_alpha"].double().cpu().numpy()
        # Gaussian id -> batch rank (projection preserves source order);
        # a SplatBatch input is indexed by rank already
        rank = spl if src is None else np.searchsorted(src, spl)
        recs = []
        for y in range(cam.height):
            row = []
            for x in range(cam.width):
                n = int(cnt[y, x])
                row.append(PixelRecords(rank[y, x, :n].astype(np.int64), tt[y, x, :n].copy(),
                                        aa[y, x, :n].copy()))
            recs.append(row)
        return recs


def _scene_for(scene, device):
    """Device copy of the scene for one call.  No implicit cache: the
    reference re-projects its (mutable) Gaussian3D list on every call, so a
    list or array dict is uploaded per call; pass a GaussianScene (or use a
    Renderer) to keep a scene resident across calls."""
    if isinstance(scene, (GaussianScene, BatchScene)):
        return scene
    if _is_batch(scene):
        return BatchScene(scene, device)
    return GaussianScene.from_any(scene, device)


def render(scene, cam: Camera, mode=None, cfg: RenderConfig | None = None, *,
           device_output: bool = False, device=None, sort_error: bool = False) -> FrameOutput:
    """Drop-in ``render`` (rasterizer.py:595-698): every sort mode, default
    FullPerPixel like the reference (rasterizer.py:598); the paper's hot
    path is ``mode=Hierarchical()``.

    ``scene`` is a list of Gaussian3D, a dict of arrays/tensors in the drop-in
    layout, a GaussianScene, or an already-projected SplatBatch.  Returns
    float64 numpy arrays like the reference unless ``device_output`` (float32
    device tensors)."""
    mode = mode if mode is not None else FullPerPixel()
    cfg = cfg or RenderConfig()
    validate_mode(mode)
    _check_supported(mode)
    dev = _require_cuda(device)
    gs = _scene_for(scene, dev)
    r = Renderer(gs, mode, cfg, dev)
    ws = workspace_for(dev)
    r.ws = ws
    return r.frame(cam, device_output=device_output, sort_error=sort_error)


def render_depth(scene, cam, mode=None, cfg: RenderConfig | None = None, **kw) -> FrameOutput:
    """rasterizer.py:701-715 (default mode FullPerPixel, :704)."""
    cfg = replace(cfg or RenderConfig(), with_depth=True)
    return render(scene, cam, mode, cfg, **kw)


def render_trajectory(scene, cameras, mode=None, cfg: RenderConfig | None = None,
                      interpolate: int = 0, **kw) -> list:
    """rasterizer.py:758-772 (default mode FullPerPixel, :761).  The scene is
    uploaded once for the whole trajectory.  Interpolation of poses is host
    logic; only ``interpolate=0`` is supported here."""
    if interpolate:
        raise ConfigError("camera interpolation is not part of the B200 path")
    dev = _require_cuda(kw.get("device"))
    gs = _scene_for(scene, dev)
    frames = []
    for i, cam in enumerate(cameras):
        try:
            frames.append(render(gs, cam, mode, cfg, **kw))
        except Exception as exc:
            raise DataError(f"frame {i}: {exc}") from exc
    return frames


@dataclass
class SortErrorStats:
    """metrics.py:37-43: out-of-order blend-depth mass per pixel."""

    delta_max: float
    delta_avg: float
    per_pixel: np.ndarray


def sort_error(frame) -> SortErrorStats:
    """metrics.sort_error (metrics.py:46-73): the per-pixel sum of positive
    depth inversions between consecutive blended contributions.  Uses the
    map the GPU accumulated during the blend (render(..., sort_error=True)),
    else the frame's blend records as the reference does."""
    if isinstance(frame, FrameOutput) and frame.sort_error is not None:
        pp = frame.sort_error
        pp = pp.double().cpu().numpy() if hasattr(pp, "cpu") else np.asarray(pp, dtype=np.float64)
    else:
        recs = frame.records if isinstance(frame, FrameOutput) else frame
        if recs is None:
            raise ConfigError("sort_error needs blend records or render(..., sort_error=True)")
        h = len(recs)
        w = len(recs[0]) if h else 0
        pp = np.zeros((h, w))
        for y in range(h):
            for x in range(w):
                d = np.asarray(recs[y][x].depth, dtype=np.float64)
                if len(d) > 1:
                    g = d[:-1] - d[1:]
                    pp[y, x] = g[g > 0].sum()
    return SortErrorStats(delta_max=float(pp.max()) if pp.size else 0.0,
                          delta_avg=float(pp.mean()) if pp.size else 0.0, per_pixel=pp)
