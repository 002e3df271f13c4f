"""View-consistency evaluation (consistency.py; the reference's
metrics.py:80-255) against a fixture the reference produced itself
(tests/golden/make_golden.py, job "consistency"): three depth frames of a
yaw sweep, its analytic flows, warp, occlusion mask and the squared-error
consistency score.  Runs on CPU tensors (the same torch code runs on the
device)."""

import os

import numpy as np
import pytest

from paper_2402_00525_b200 import Camera, ConfigError, FrameOutput
from paper_2402_00525_b200 import consistency as C

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def fx():
    z = np.load(os.path.join(G, "io_consistency.npz"))
    d = {k: z[k] for k in z.files}
    frames = [FrameOutput(color=d[f"color{k}"], transmittance=d[f"tn{k}"], depth=d[f"depth{k}"])
              for k in range(3)]
    cams = [Camera(rotation=d[f"R{k}"], position=d[f"pos{k}"], fx=80.0, fy=80.0, width=96,
                   height=72) for k in range(3)]
    return d, frames, cams


def test_analytic_flow(fx):
    d, frames, cams = fx
    for i in range(3):
        for j in range(3):
            if i == j:
                continue
            fl, va = C.analytic_flow(frames[i], cams[i], cams[j])
            np.testing.assert_array_equal(va.numpy(), d[f"valid{i}{j}"])
            np.testing.assert_allclose(fl.numpy(), d[f"flow{i}{j}"], rtol=1e-9, atol=1e-9)


def test_warp_and_occlusion(fx):
    d, frames, cams = fx
    wa, wv = C.warp_frame(d["color1"], d["flow01"])
    np.testing.assert_array_equal(wv.numpy(), d["warpvalid01"])
    np.testing.assert_allclose(wa.numpy(), d["warp01"], rtol=1e-12, atol=1e-12)
    occ = C.occlusion_mask(d["flow01"], d["flow10"])
    np.testing.assert_array_equal(occ.numpy(), d["occ01"])


def test_view_consistency_mse(fx):
    d, frames, cams = fx
    fw = {(i, j): (d[f"flow{i}{j}"], d[f"valid{i}{j}"]) for i in range(3) for j in range(3)
          if j > i}
    bw = {(i, j): (d[f"flow{i}{j}"], d[f"valid{i}{j}"]) for i in range(3) for j in range(3)
          if j < i}
    rep = C.view_consistency(frames, fw, bw, offsets=(1, 2), metric="both", crop=4)
    np.testing.assert_allclose([rep.mse_t[1], rep.mse_t[2]], d["mse_t"], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose([rep.flip_t[1], rep.flip_t[2]], d["flip_t"], rtol=1e-7,
                               atol=1e-12)
    with pytest.raises(ConfigError):
        C.view_consistency(frames, fw, bw, metric="psnr")
    with pytest.raises(ConfigError):
        C.view_consistency(frames, fw, bw, offsets=(5,))


def test_flip_error_map(fx):
    """flip.flip_error_map (colour + feature pipelines) == the reference's
    map for frame 0 against frame 1 warped onto it; symmetric, zero on
    identical inputs."""
    d, frames, cams = fx
    m = C.flip_error_map(d["color0"], d["warp01"]).numpy()
    np.testing.assert_allclose(m, d["flip01"], rtol=1e-7, atol=1e-9)
    m2 = C.flip_error_map(d["warp01"], d["color0"]).numpy()
    np.testing.assert_allclose(m, m2, rtol=1e-12, atol=1e-12)
    assert float(C.flip_error_map(d["color0"], d["color0"]).abs().max()) == 0.0
