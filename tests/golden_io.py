"""Load the committed golden fixtures (tests/golden/*.npz, produced by the
reference package via tests/golden/make_golden.py) into framework objects."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

from paper_2402_00525_b200.types import (Camera, FullPerPixel, GlobalZ, Hierarchical,
                                         RenderConfig, Window)

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith(("grad_", "io_")))


def grad_names():
    """Fixtures with reference gradients (grad_<name>.npz)."""
    return sorted(os.path.basename(p)[5:-4]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "grad_*.npz")))


def load_grad(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"grad_{name}.npz"))
    return {k: z[k] for k in z.files}


def load(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    d = {k: z[k] for k in z.files}
    fx, fy, cx, cy = d["cam_intr"]
    w, h = (int(v) for v in d["cam_size"])
    cam = Camera(rotation=d["cam_R"], position=d["cam_pos"], fx=fx, fy=fy, width=w, height=h,
                 cx=cx, cy=cy)
    cfg_d = json.loads(str(d["cfg_json"]))
    cfg = RenderConfig(**cfg_d)
    md = json.loads(str(d["mode_json"]))
    kind = md.pop("mode", "hierarchical")
    mode = {"globalz": GlobalZ, "full": FullPerPixel}.get(kind)
    mode = mode() if mode else (Window(**md) if kind == "window" else Hierarchical(**md))
    scene = {k: d[k] for k in ("means", "quats", "scales", "opacity", "sh")}
    return scene, cam, cfg, mode, d


def records_of(d, i):
    """(splat, t, alpha) of the i-th recorded pixel."""
    a, b = int(d["rec_offsets"][i]), int(d["rec_offsets"][i + 1])
    return d["rec_splat"][a:b], d["rec_t"][a:b], d["rec_alpha"][a:b]
