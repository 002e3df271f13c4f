"""The drop-in shim (paper_2402_00525_b200.splatsort_plugin)
on the reference package installed in baseline/_ref (baseline/install_ref.sh).

CPU tests: the shim rebinds exactly the reference's render entry points, maps
modes and configs, keeps the reference's error classes, and has no CPU
fallback (without a GPU every render raises instead of silently running the
reference's own renderer).  The GPU replay of the
reference's own tests through the shim is tests/test_reference_replay.py.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "splatsort")),
                                reason="reference not installed (baseline/install_ref.sh)")


@pytest.fixture()
def ss():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import splatsort
    from paper_2402_00525_b200 import splatsort_plugin as P
    P.install(splatsort)
    yield splatsort
    P.uninstall()


def test_install_rebinds_render_entry_points(ss):
    from paper_2402_00525_b200 import splatsort_plugin as P
    assert P.installed()
    for fn in (ss.rasterizer.render, ss.render, ss.gradients.render):
        assert getattr(fn, "__b200__", False)
    # render_depth / render_trajectory are the reference's own wrappers and
    # reach the B200 render through the rasterizer module global
    assert ss.rasterizer.render_depth.__module__ == "splatsort.rasterizer"
    P.uninstall()
    assert not getattr(ss.rasterizer.render, "__b200__", False)
    assert not getattr(ss.render, "__b200__", False)
    P.install(ss)


def test_mode_and_config_mapping(ss):
    from paper_2402_00525_b200 import splatsort_plugin as P
    from paper_2402_00525_b200 import types as T
    r = ss.rasterizer
    h = P._mode(r.Hierarchical(queue_tail=96, queue_mid=12, queue_head=2,
                               mid_depth_at_center=True), ss)
    assert h == T.Hierarchical(queue_tail=96, queue_mid=12, queue_head=2,
                               mid_depth_at_center=True)
    assert P._mode(r.Window(24), ss) == T.Window(24)
    assert P._mode(r.GlobalZ(), ss) == T.GlobalZ()
    assert P._mode(r.FullPerPixel(), ss) == T.FullPerPixel()
    c = P._cfg(r.RenderConfig(background=[0.1, 0.2, 0.3], with_depth=True,
                              exact_tile_culling=False, termination=1e-3), ss)
    assert isinstance(c, T.RenderConfig) and c.with_depth and c.exact_tile_culling is False
    np.testing.assert_array_equal(c.background, [0.1, 0.2, 0.3])
    assert c.termination == 1e-3


def test_reference_errors_and_no_cpu_fallback(ss):
    import torch
    r = ss.rasterizer
    cam = ss.Camera(rotation=np.eye(3), position=np.zeros(3), fx=50.0, fy=50.0, width=32,
                    height=32)
    g = ss.Gaussian3D(mean=[0, 0, 2.0], rotation=[1, 0, 0, 0], scale=[0.1] * 3, opacity=0.5,
                      sh=np.zeros((16, 3)))
    with pytest.raises(ss.errors.ConfigError):          # the reference's validate_mode
        r.render([g], cam, r.Window(0))
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the replay")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        r.render([g], cam, r.Hierarchical())
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        r.render_depth([g], cam, r.FullPerPixel())
