"""Drop the B200 render path into the reference package ``splatsort``.

This is INTEGRATION.md §1 as an importable, tested module.  ``install()``
rebinds the reference's render entry points to the B200 path:

* ``splatsort.rasterizer.render`` (rasterizer.py:595-698) -- and through the
  module global, ``render_depth`` (:701-715) and ``render_trajectory``
  (:758-772, camera interpolation stays the reference's host code);
* ``splatsort.render`` (the public re-export, __init__.py:42-61);
* ``splatsort.gradients.render`` (gradients.py:22 imports the name), so the
  reference's ``backward_render`` renders its forward pass (with records) on
  the GPU and differentiates the GPU's blend order on the host.

``splatsort.metrics`` imports ``render_depth`` by name (metrics.py:20-26); that
is the reference's own wrapper, which calls the rebound module-global
``render``, so it needs no patch.

Arguments are the reference's own objects (``Gaussian3D`` lists or a
``SplatBatch``, ``Camera``, the four sort modes, ``RenderConfig``); results
are the reference's own ``FrameOutput`` / ``PixelRecords`` classes, float64
numpy, same ``stats`` keys.  Errors keep their classes: an invalid mode or
config raises the reference's ``ConfigError`` (its own ``validate_mode`` runs
first), a per-frame failure its ``DataError``.  There is no CPU fallback:
every mode and window size renders on the device, and a missing GPU or
extension raises.

As a pytest plugin (``pytest -p paper_2402_00525_b200.splatsort_plugin``)
it installs itself before test modules are imported, so a reference test's
``from splatsort.rasterizer import render`` binds the B200 path; this is how
``tests/test_reference_replay.py`` replays the reference's own hot-path tests.
"""

from __future__ import annotations

import importlib

import numpy as np

_STATE: dict = {}


def _ours():
    from . import renderer, types
    return renderer, types


def _mode(mode, ss):
    """reference SortMode -> this package's (rasterizer.py:47-89)."""
    _, T = _ours()
    r = ss.rasterizer
    if isinstance(mode, r.Hierarchical):
        return T.Hierarchical(queue_tail=mode.queue_tail, queue_mid=mode.queue_mid,
                              queue_head=mode.queue_head, batch_load=mode.batch_load,
                              batch_mid=mode.batch_mid, batch_head=mode.batch_head,
                              mid_depth_at_center=mode.mid_depth_at_center)
    if isinstance(mode, r.Window):
        return T.Window(mode.size)
    if isinstance(mode, r.GlobalZ):
        return T.GlobalZ()
    if isinstance(mode, r.FullPerPixel):
        return T.FullPerPixel()
    raise ss.errors.ConfigError(f"unknown sort mode {mode!r}")


def _cfg(cfg, ss):
    _, T = _ours()
    if cfg is None:
        return None
    return T.RenderConfig(
        tile_size=cfg.tile_size, opacity_eps=cfg.opacity_eps, termination=cfg.termination,
        alpha_cap=cfg.alpha_cap, background=np.asarray(cfg.background, dtype=np.float64),
        near=cfg.near, guard_band=cfg.guard_band, dilation=cfg.dilation,
        inv_scale_clamp=cfg.inv_scale_clamp, capture_records=cfg.capture_records,
        with_depth=cfg.with_depth, workers=cfg.workers,
        exact_tile_culling=cfg.exact_tile_culling)


def _frame(out, ss):
    """this package's FrameOutput -> the reference's (rasterizer.py:234-255)."""
    r = ss.rasterizer
    recs = None
    if out.records is not None:
        recs = [[r.PixelRecords(np.asarray(p.splat, dtype=np.int64),
                                np.asarray(p.depth, dtype=np.float64),
                                np.asarray(p.alpha, dtype=np.float64)) for p in row]
                for row in out.records]
    stats = dict(out.stats)
    stats.pop("tie_runs", None)          # B200-only diagnostic, not a reference key
    return r.FrameOutput(color=out.color, transmittance=out.transmittance, depth=out.depth,
                         records=recs,
                         source_index=np.asarray(out.source_index, dtype=np.int64).copy(),
                         stats=stats)


def make_render(ss):
    """The B200 ``render`` with the reference signature (rasterizer.py:595-600)."""
    renderer, T = _ours()
    r = ss.rasterizer

    def render(scene, cam, mode=r.FullPerPixel(), cfg=None):
        r.validate_mode(mode)                  # the reference's ConfigError, its messages
        _STATE["calls"] = _STATE.get("calls", 0) + 1
        m = _mode(mode, ss)
        c = _cfg(cfg, ss)
        if isinstance(scene, ss.gaussian_math.SplatBatch) and len(scene) == 0:
            scene = []                         # an empty batch renders the background
        try:
            out = renderer.render(scene, cam, m, c)
        except T.ConfigError as exc:
            raise ss.errors.ConfigError(str(exc)) from exc
        except T.DataError as exc:
            raise ss.errors.DataError(str(exc)) from exc
        return _frame(out, ss)

    render.__doc__ = "B200 render (paper_2402_00525_b200.splatsort_plugin)"
    render.__b200__ = True
    return render


def install(ss=None):
    """Rebind the reference's render entry points to the B200 path.
    Idempotent; returns the ``splatsort`` module."""
    if ss is None:
        ss = importlib.import_module("splatsort")
    for sub in ("rasterizer", "gradients", "metrics", "gaussian_math", "errors"):
        importlib.import_module(f"splatsort.{sub}")
    if _STATE.get("module") is ss:
        return ss
    fn = make_render(ss)
    saved = {
        (ss.rasterizer, "render"): ss.rasterizer.render,
        (ss, "render"): ss.render,
        (ss.gradients, "render"): ss.gradients.render,
    }
    ss.rasterizer.render = fn
    ss.render = fn
    ss.gradients.render = fn
    _STATE.update(module=ss, saved=saved)
    return ss


def uninstall():
    ss = _STATE.pop("module", None)
    for (mod, name), fn in _STATE.pop("saved", {}).items():
        setattr(mod, name, fn)
    return ss


def installed() -> bool:
    return "module" in _STATE


# ---------------------------------------------------------------------------
# pytest plugin: `pytest -p paper_2402_00525_b200.splatsort_plugin`

def pytest_configure(config):
    install()


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    import torch
    terminalreporter.write_line(
        f"splatsort_plugin: {_STATE.get('calls', 0)} render calls on the B200 path "
        f"({torch.cuda.get_device_name(0) if torch.cuda.is_available() else 'no GPU'})")
