"""Small renders of every K6 variant and the sort for compute-sanitizer
(scripts/sanitize.sh runs this under memcheck, racecheck, synccheck and
initcheck).  C1 (10k Gaussians, 256x256) plus a 20k C3-layout view with
depth, records, sort error, float64 outputs and the backward replay."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_00525_b200 import (FullPerPixel, GlobalZ, Hierarchical, RenderConfig,  # noqa
                                   Window, backward_render, scenes)
from paper_2402_00525_b200.renderer import Renderer  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
sc, cams = scenes.config_scene("C1")
garden = scenes.to_f32_scene(scenes.garden_scene(20_000, 3))
gcam = scenes.orbit_cameras(8, width=256, height_px=144, f=146.0)[6]
modes = [Hierarchical(), Hierarchical(queue_tail=96, queue_mid=12, queue_head=2), GlobalZ(),
         FullPerPixel(), Window(8), Window(24)]
if which != "all":
    modes = [m for m in modes if type(m).__name__.lower().startswith(which)]
for m in modes:
    r = Renderer(sc, m, RenderConfig())
    out = r.frame(cams[0])
    r2 = Renderer(garden, m, RenderConfig(with_depth=True, capture_records=True))
    out2 = r2.frame(gcam, sort_error=True)
    outs = r2.alloc_outputs(gcam.width, gcam.height)
    r2.render_into(gcam, outs)                      # the asynchronous (benched) call
    torch.cuda.synchronize()
    assert r2.check_status()
    print(f"{type(m).__name__:13s} C1 entries {out.stats['bin_entries']:7d}  garden entries "
          f"{out2.stats['bin_entries']:7d}  mean colour {float(np.mean(out2.color)):.5f}",
          flush=True)
up = np.random.default_rng(0).normal(0, 1, (gcam.height, gcam.width, 3))
g = backward_render(garden, gcam, Hierarchical(), up, RenderConfig())
print("backward |d_color|", float(np.abs(g.d_color).sum()), flush=True)
print("sanitize driver done", flush=True)
