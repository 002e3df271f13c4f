"""Plain-render K6 time of Window(k) on C3 views (the register window vs the
shared-memory heap kernel; STP_LIB_VARIANT selects a build).
usage: python scripts/window_timing.py [k ...]   (0 = FullPerPixel, -1 = GlobalZ)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_00525_b200 import FullPerPixel, GlobalZ, RenderConfig, Window, scenes  # noqa: E402
from paper_2402_00525_b200.renderer import Renderer  # noqa: E402

ks = [int(a) for a in sys.argv[1:]] or [3, 4, 8, 12, 16, 24]   # 0 = FullPerPixel, -1 = GlobalZ
sc, cams = scenes.config_scene("C3")
for k in ks:
    mode = GlobalZ() if k < 0 else (Window(k) if k else FullPerPixel())
    r = Renderer(sc, mode, RenderConfig())
    outs = r.alloc_outputs(cams[0].width, cams[0].height)
    r.render_into(cams[0], outs, stats=True, timings=True)
    ms = [r.render_into(cams[v], outs, stats=True, timings=True).ms_blend for v in (0, 64, 128)]
    print(json.dumps({"window": k, "ms_render": float(np.mean(ms)),
                      "variant": os.environ.get("STP_LIB_VARIANT", "default")}), flush=True)
