"""CPU checks of the drop-in boundary (no GPU needed, no compute calls).

* libstp_b200.so loads and exports every function include/stp.h declares;
* the ctypes struct mirrors have the C sizes the header implies;
* host-only entry points (version, error strings, config validation,
  workspace sizing / layout) behave like the reference's validate_mode /
  RenderConfig checks (rasterizer.py:93-117, 196-203).
"""

import ctypes
import os
import re

import pytest

from paper_2402_00525_b200 import (ConfigError, FullPerPixel, Hierarchical, RenderConfig,
                                   _lib, parse_mode, validate_mode)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stp.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(stp_\w+)\s*\(", src,
                                 flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_header_declares_the_abi():
    fns = declared_functions()
    assert "stp_render" in fns and "stp_workspace_bytes" in fns and len(fns) >= 10


def test_library_exports_every_declared_symbol(lib):
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert set(declared_functions()) == set(_lib.EXPORTS)


def test_struct_layouts_match_header(tmp_path):
    """Compile a probe against include/stp.h and compare every struct's size
    and field offsets with the ctypes mirrors."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"StpScene": _lib.StpScene, "StpSplatBatch": _lib.StpSplatBatch,
               "StpCamera": _lib.StpCamera,
               "StpConfig": _lib.StpConfig, "StpOutputs": _lib.StpOutputs,
               "StpStats": _lib.StpStats, "StpLayout": _lib.StpLayout}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "stp.h"', 'int main(void){']
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def test_version_and_errors(lib):
    assert lib.stp_abi_version() == _lib.ABI_VERSION == 3
    assert _lib.error_string(_lib.STP_OK) == "ok"
    assert "configuration" in _lib.error_string(_lib.STP_ERR_CONFIG)
    assert "workspace" in _lib.error_string(_lib.STP_ERR_WORKSPACE_TOO_SMALL)
    assert lib.stp_error_string(99) == b"unknown error"


def _cfg(mode=None, cfg=None):
    from paper_2402_00525_b200.renderer import make_config
    return make_config(cfg or RenderConfig(), mode or Hierarchical())


def test_validate_config_accepts_defaults(lib):
    assert lib.stp_validate_config(ctypes.byref(_cfg())) == _lib.STP_OK
    for qh in (1, 2, 4, 8, 16):
        c = _cfg(Hierarchical(queue_head=qh))
        assert lib.stp_validate_config(ctypes.byref(c)) == _lib.STP_OK
    c = _cfg(Hierarchical(queue_tail=128, queue_mid=16))
    assert lib.stp_validate_config(ctypes.byref(c)) == _lib.STP_OK


@pytest.mark.parametrize("field,value", [
    ("q_tail", 48), ("q_tail", 80), ("q_mid", 6), ("q_head", 0), ("tile_size", 8),
    ("b_load", 16), ("b_mid", 8), ("b_head", 2), ("q_tail", 512), ("record_cap", -1)])
def test_validate_config_rejects(lib, field, value):
    c = _cfg()
    setattr(c, field, value)
    assert lib.stp_validate_config(ctypes.byref(c)) == _lib.STP_ERR_CONFIG


def test_validate_config_modes_and_bands(lib):
    """Sort modes (GlobalZ / FullPerPixel / Window <= 512) and K6 tile bands
    through the host-side config check (no device work)."""
    from paper_2402_00525_b200 import FullPerPixel, GlobalZ, Window
    from paper_2402_00525_b200.renderer import make_config
    for m in (GlobalZ(), FullPerPixel(), Window(1), Window(8), Window(16), Window(17), Window(512)):
        c = make_config(RenderConfig(), m)
        assert lib.stp_validate_config(ctypes.byref(c)) == _lib.STP_OK, m
    c = make_config(RenderConfig(), Window(513))
    assert lib.stp_validate_config(ctypes.byref(c)) == _lib.STP_ERR_CONFIG
    c = _cfg()
    c.sort_mode = 7
    assert lib.stp_validate_config(ctypes.byref(c)) == _lib.STP_ERR_CONFIG
    for band, ok in (((0, 10), True), ((5, 5), False), ((-1, 4), False), ((0, 0), True)):
        c = make_config(RenderConfig(), Hierarchical(), tiles=band)
        want = _lib.STP_OK if ok else _lib.STP_ERR_CONFIG
        assert lib.stp_validate_config(ctypes.byref(c)) == want, band


def test_validate_config_alpha_cap(lib):
    c = _cfg()
    for bad in (0.0, 1.0, 1.5):
        c.alpha_cap = bad
        assert lib.stp_validate_config(ctypes.byref(c)) == _lib.STP_ERR_CONFIG


def test_workspace_layout(lib):
    n, W, H = 1000, 1920, 1080
    b0 = lib.stp_workspace_bytes(n, W, H, 0)
    b1 = lib.stp_workspace_bytes(n, W, H, 100_000)
    assert 0 < b0 < b1
    assert lib.stp_workspace_bytes(-1, W, H, 0) == 0
    L = _lib.StpLayout()
    assert lib.stp_workspace_layout(n, W, H, b1, ctypes.byref(L)) == _lib.STP_OK
    assert L.entry_capacity >= 100_000 and L.total <= b1
    assert (L.grid_w, L.grid_h, L.n_tiles) == (120, 68, 8160)
    # 13 tile bits + 27 depth bits: 5 eight-bit passes; ids in the low 10 bits
    assert (L.sort_bits, L.depth_bits, L.sort_passes, L.id_bits) == (40, 27, 5, 10)
    regions = sorted((getattr(L, k), k) for k in ("recs", "camera", "masks",
                                                    "state", "counts", "offsets", "keys0",
                                                    "keys1", "vals", "ranges",
                                                    "counters", "hist", "lookback",
                                                    "scan_scratch"))
    offs = [o for o, _ in regions]
    assert len(set(offs)) == len(offs) and all(o % 256 == 0 for o in offs)
    # every region holds what its kernels write: K2's block partials (one per
    # 4096 counts, + 1), the per-Gaussian arrays, the ping-pong key buffers
    size = {k: (regions[i + 1][0] if i + 1 < len(regions) else L.total) - o
            for i, (o, k) in enumerate(regions)}
    for nn in (1000, 4095, 4097, 3_000_000):
        Ln = _lib.StpLayout()
        bn = lib.stp_workspace_bytes(nn, W, H, 1000)
        assert lib.stp_workspace_layout(nn, W, H, bn, ctypes.byref(Ln)) == _lib.STP_OK
        rn = sorted((getattr(Ln, k), k) for k in ("recs", "camera", "masks", "state", "counts",
                                                   "offsets", "keys0", "keys1", "vals", "ranges",
                                                   "counters", "hist", "lookback",
                                                   "scan_scratch"))
        sz = {k: (rn[i + 1][0] if i + 1 < len(rn) else Ln.total) - o
              for i, (o, k) in enumerate(rn)}
        assert sz["scan_scratch"] >= ((nn + 4095) // 4096 + 1) * 4
        assert sz["counts"] >= 4 * nn and sz["offsets"] >= 4 * nn
        assert sz["keys0"] >= 8 * Ln.entry_capacity and sz["vals"] >= 4 * Ln.entry_capacity
    assert size["recs"] >= 160 * n
    assert lib.stp_workspace_layout(n, W, H, 16, ctypes.byref(L)) == \
        _lib.STP_ERR_WORKSPACE_TOO_SMALL
    # 4K frame: 32,400 tiles -> 47-bit keys
    b = lib.stp_workspace_bytes(n, 3840, 2160, 1000)
    assert lib.stp_workspace_layout(n, 3840, 2160, b, ctypes.byref(L)) == _lib.STP_OK
    assert L.n_tiles == 32400 and (L.sort_bits, L.depth_bits) == (40, 25)
    # 6M Gaussians at 4K: 23 id bits, 15 tile + 25 depth bits = 63
    b = lib.stp_workspace_bytes(6_000_000, 3840, 2160, 1000)
    assert lib.stp_workspace_layout(6_000_000, 3840, 2160, b, ctypes.byref(L)) == _lib.STP_OK
    assert (L.id_bits, L.sort_bits, L.sort_passes) == (23, 40, 5)
    # 100M Gaussians: the word keeps 64 - 27 = 37 key bits (22 depth bits)
    b = lib.stp_workspace_bytes(100_000_000, 3840, 2160, 1000)
    assert lib.stp_workspace_layout(100_000_000, 3840, 2160, b, ctypes.byref(L)) == _lib.STP_OK
    assert (L.id_bits, L.sort_bits, L.depth_bits) == (27, 37, 22)


def test_host_mode_validation_mirrors_reference():
    validate_mode(Hierarchical())
    with pytest.raises(ConfigError):
        validate_mode(Hierarchical(queue_tail=48))
    with pytest.raises(ConfigError):
        validate_mode(Hierarchical(queue_mid=6))
    assert isinstance(parse_mode("hierarchical"), Hierarchical)
    assert isinstance(parse_mode("full"), FullPerPixel)
    with pytest.raises(ConfigError):
        parse_mode("nonsense")


def test_product_path_has_no_cpu_fallback():
    """Without a CUDA device the product entry points raise instead of
    computing on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2402_00525_b200 import render
    from paper_2402_00525_b200.types import Camera
    import numpy as np
    cam = Camera(rotation=np.eye(3), position=np.zeros(3), fx=100.0, fy=100.0, width=32,
                 height=32)
    scene = {"means": np.zeros((1, 3)), "quats": np.array([[1.0, 0, 0, 0]]),
             "scales": np.ones((1, 3)) * 0.1, "opacity": np.ones(1) * 0.5,
             "sh": np.zeros((1, 1, 3))}
    with pytest.raises(RuntimeError, match="CUDA"):
        render(scene, cam, Hierarchical())


def test_product_modules_do_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2402_00525_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s, f
                assert "libstp_oracle" not in s, f
