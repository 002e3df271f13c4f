"""ctypes binding of the C ABI in include/stp.h (libstp_b200.so, built in-tree).

The product path fails loudly when the library is missing or no CUDA device
is present: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstp_b200.so")

STP_OK, STP_ERR_CONFIG, STP_ERR_DATA, STP_ERR_WORKSPACE_TOO_SMALL, STP_ERR_CUDA = range(5)
STP_FLAG_TIMINGS = 1
STP_STAGE_EVENTS = 5    # [K0+K1 | K2+K3 | K4+K5 | K6]
STP_KERNEL_EVENTS = 8   # [K0 | K1 | K2 | K3 | K4 | K5 | K6]
ABI_VERSION = 3
STP_MODE_HIERARCHICAL = 0
STP_MODE_GLOBALZ = 1
STP_MODE_FULL = 2
STP_MODE_WINDOW = 3

EXPORTS = ("stp_abi_version", "stp_error_string", "stp_validate_config", "stp_workspace_bytes",
           "stp_workspace_layout", "stp_render", "stp_render_batch", "stp_render_views",
           "stp_read_stats",
           "stp_render_events", "stp_events_create", "stp_events_destroy",
           "stp_event_elapsed_ms", "stp_backward", "stp_backward_batch")


class StpScene(ctypes.Structure):
    _fields_ = [("means", ctypes.c_void_p), ("quats", ctypes.c_void_p),
                ("scales", ctypes.c_void_p), ("opacity", ctypes.c_void_p),
                ("sh", ctypes.c_void_p), ("n", ctypes.c_int64), ("sh_coeffs", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class StpSplatBatch(ctypes.Structure):
    _fields_ = [("mean2d", ctypes.c_void_p), ("conic", ctypes.c_void_p),
                ("color", ctypes.c_void_p), ("opacity", ctypes.c_void_p),
                ("radius", ctypes.c_void_p), ("inv_cov3", ctypes.c_void_p),
                ("inv_cov_center", ctypes.c_void_p), ("n", ctypes.c_int64),
                ("global_depth", ctypes.c_void_p), ("center_dist", ctypes.c_void_p)]


class StpCamera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("pos", ctypes.c_double * 3),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class StpConfig(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("termination", ctypes.c_double),
                ("alpha_cap", ctypes.c_double), ("bg", ctypes.c_double * 3),
                ("near_plane", ctypes.c_double), ("guard", ctypes.c_double),
                ("dilation", ctypes.c_double), ("inv_scale_clamp", ctypes.c_double),
                ("tile_size", ctypes.c_int32), ("q_tail", ctypes.c_int32),
                ("q_mid", ctypes.c_int32), ("q_head", ctypes.c_int32),
                ("b_load", ctypes.c_int32), ("b_mid", ctypes.c_int32),
                ("b_head", ctypes.c_int32), ("mid_depth_at_center", ctypes.c_int32),
                ("with_depth", ctypes.c_int32), ("exact_culling", ctypes.c_int32),
                ("record_cap", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("sort_mode", ctypes.c_int32), ("tile_begin", ctypes.c_int32),
                ("tile_end", ctypes.c_int32)]


class StpOutputs(ctypes.Structure):
    _fields_ = [("color", ctypes.c_void_p), ("transmittance", ctypes.c_void_p),
                ("depth", ctypes.c_void_p), ("rec_count", ctypes.c_void_p),
                ("rec_splat", ctypes.c_void_p), ("rec_t", ctypes.c_void_p),
                ("rec_alpha", ctypes.c_void_p), ("state", ctypes.c_void_p),
                ("sort_error", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("color64", ctypes.c_void_p), ("transmittance64", ctypes.c_void_p),
                ("depth64", ctypes.c_void_p), ("rec_t64", ctypes.c_void_p),
                ("rec_alpha64", ctypes.c_void_p), ("splat_color64", ctypes.c_void_p)]


class StpGrads(ctypes.Structure):
    _fields_ = [("upstream", ctypes.c_void_p), ("pix_state", ctypes.c_void_p),
                ("d_color", ctypes.c_void_p), ("d_opacity", ctypes.c_void_p),
                ("d_mean2d", ctypes.c_void_p), ("d_conic", ctypes.c_void_p)]


class StpStats(ctypes.Structure):
    _fields_ = [("input", ctypes.c_int64), ("behind", ctypes.c_int64),
                ("guard", ctypes.c_int64), ("degenerate", ctypes.c_int64),
                ("kept", ctypes.c_int64), ("bin_entries", ctypes.c_int64),
                ("tiles", ctypes.c_int64), ("nonfinite_pixels", ctypes.c_int64),
                ("tie_runs", ctypes.c_int64), ("entry_capacity", ctypes.c_int64),
                ("ms_project", ctypes.c_float), ("ms_duplicate", ctypes.c_float),
                ("ms_sort", ctypes.c_float), ("ms_blend", ctypes.c_float),
                ("ms_total", ctypes.c_float), ("overflow", ctypes.c_int32)]


class StpLayout(ctypes.Structure):
    _fields_ = [(n, ctypes.c_size_t) for n in (
        "recs", "camera", "masks", "state", "counts", "offsets", "keys0", "keys1", "vals", "ranges",
        "counters", "hist", "lookback", "scan_scratch", "rowlist", "aux", "total")] + [
        ("entry_capacity", ctypes.c_int64), ("n_tiles", ctypes.c_int32),
        ("grid_w", ctypes.c_int32), ("grid_h", ctypes.c_int32),
        ("sort_passes", ctypes.c_int32), ("sort_bits", ctypes.c_int32),
        ("partitions", ctypes.c_int32), ("splat_record_bytes", ctypes.c_int32),
        ("final_buffer", ctypes.c_int32), ("depth_bits", ctypes.c_int32),
        ("id_bits", ctypes.c_int32)]


_lib = None


def load(build_if_missing: bool = True):
    """Load libstp_b200.so (building it with nvcc if absent or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    # A/B experiments (scripts/ab.sh): an alternative in-tree build of the
    # same sources with different compile-time knobs
    path = os.environ.get("STP_LIB_VARIANT") or LIB_PATH
    if path == LIB_PATH and build_if_missing and _build.needs_build():
        _build.build()
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run paper_2402_00525_b200/build.py "
                           "(no CPU fallback exists)")
    L = ctypes.CDLL(path)
    L.stp_abi_version.restype = ctypes.c_int
    L.stp_error_string.restype = ctypes.c_char_p
    L.stp_error_string.argtypes = [ctypes.c_int]
    L.stp_validate_config.argtypes = [ctypes.POINTER(StpConfig)]
    L.stp_workspace_bytes.restype = ctypes.c_size_t
    L.stp_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int64]
    L.stp_workspace_layout.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_size_t, ctypes.POINTER(StpLayout)]
    L.stp_render.argtypes = [ctypes.POINTER(StpScene), ctypes.POINTER(StpCamera),
                             ctypes.POINTER(StpConfig), ctypes.c_void_p, ctypes.c_size_t,
                             ctypes.POINTER(StpOutputs), ctypes.POINTER(StpStats),
                             ctypes.c_void_p]
    for fn, sc in (("stp_backward", StpScene), ("stp_backward_batch", StpSplatBatch)):
        getattr(L, fn).argtypes = [ctypes.POINTER(sc), ctypes.POINTER(StpCamera),
                                   ctypes.POINTER(StpConfig), ctypes.c_void_p, ctypes.c_size_t,
                                   ctypes.POINTER(StpOutputs), ctypes.POINTER(StpGrads),
                                   ctypes.c_void_p, ctypes.c_void_p]
    L.stp_render_batch.argtypes = [ctypes.POINTER(StpSplatBatch), ctypes.POINTER(StpCamera),
                                   ctypes.POINTER(StpConfig), ctypes.c_void_p, ctypes.c_size_t,
                                   ctypes.POINTER(StpOutputs), ctypes.POINTER(StpStats),
                                   ctypes.c_void_p]
    L.stp_render_views.argtypes = [ctypes.POINTER(StpScene), ctypes.POINTER(StpCamera),
                                   ctypes.c_int32, ctypes.POINTER(StpConfig), ctypes.c_void_p,
                                   ctypes.c_size_t, ctypes.POINTER(StpOutputs), ctypes.c_void_p]
    L.stp_read_stats.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64,
                                 ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(StpStats),
                                 ctypes.c_void_p]
    L.stp_render_events.argtypes = [ctypes.POINTER(StpScene), ctypes.POINTER(StpCamera),
                                    ctypes.POINTER(StpConfig), ctypes.c_void_p,
                                    ctypes.c_size_t, ctypes.POINTER(StpOutputs),
                                    ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                    ctypes.c_void_p]
    L.stp_events_create.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]
    L.stp_events_destroy.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]
    L.stp_event_elapsed_ms.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.POINTER(ctypes.c_float)]
    if L.stp_abi_version() != ABI_VERSION:
        raise RuntimeError("libstp_b200.so ABI version mismatch")
    _lib = L
    return L


def error_string(code: int) -> str:
    return load().stp_error_string(code).decode()
