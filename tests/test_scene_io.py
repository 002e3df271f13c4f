"""Scene / camera input against files written by the
reference itself (tests/golden/make_golden.py, job "io"): the decoded arrays
equal what the reference's own loaders return; malformed files raise
SceneFormatError like scene_io.py:152-254, 366-417.  CPU only."""

import os

import numpy as np
import pytest

from paper_2402_00525_b200 import SceneFormatError
from paper_2402_00525_b200.scene_io import load_cameras, load_ply, load_ply_arrays

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PLY = os.path.join(G, "io_cloud200.ply")


def _expected():
    z = np.load(os.path.join(G, "io_expected.npz"))
    return {k: z[k] for k in z.files}


def test_ply_matches_reference_loader():
    a, e = load_ply_arrays(PLY), _expected()
    for k in ("means", "quats", "scales", "opacity", "sh"):
        assert a[k].dtype == np.float32 and a[k].flags.c_contiguous
        np.testing.assert_allclose(a[k], e[k], rtol=1e-6, atol=1e-7, err_msg=k)
    assert a["sh"].shape == (200, 16, 3)
    gs = load_ply(PLY)
    assert len(gs) == 200
    np.testing.assert_allclose(gs[7].sh, e["sh"][7], rtol=1e-6, atol=1e-7)


def test_cameras_match_reference_loader():
    cams, e = load_cameras(os.path.join(G, "io_cams.json")), _expected()
    assert len(cams) == len(e["cam_R"])
    for c, R, p, intr, size in zip(cams, e["cam_R"], e["cam_pos"], e["cam_intr"], e["cam_size"]):
        np.testing.assert_allclose(c.rotation, R, atol=1e-12)
        np.testing.assert_allclose(c.position, p)
        np.testing.assert_allclose([c.fx, c.fy, c.cx, c.cy], intr)
        assert [c.width, c.height] == size.tolist()


def test_malformed_files_raise(tmp_path):
    raw = open(PLY, "rb").read()
    bad = {
        "trunc": raw[:-100],
        "noend": raw.replace(b"end_header", b"end_hXader"),
        "ascii": raw.replace(b"binary_little_endian", b"ascii"),
        "missing": raw.replace(b"property float rot_3", b"property float rot_9"),
        "notply": b"plx" + raw[3:],
    }
    for name, b in bad.items():
        p = tmp_path / f"{name}.ply"
        p.write_bytes(b)
        with pytest.raises(SceneFormatError):
            load_ply_arrays(p)
    cj = tmp_path / "c.json"
    cj.write_text('[{"width": 4, "height": 4, "position": [0,0,0], '
                  '"rotation": [[1,0,0],[0,1,0],[0,0,2]], "fx": 1, "fy": 1}]')
    with pytest.raises(SceneFormatError):
        load_cameras(cj)
    cj.write_text('{"not": "a list"}')
    with pytest.raises(SceneFormatError):
        load_cameras(cj)


def test_non_finite_record_raises(tmp_path):
    raw = bytearray(open(PLY, "rb").read())
    off = raw.find(b"end_header") + len(b"end_header\n")
    raw[off:off + 4] = np.float32(np.nan).tobytes()   # x of record 0
    p = tmp_path / "nan.ply"
    p.write_bytes(bytes(raw))
    with pytest.raises(SceneFormatError):
        load_ply_arrays(p)
