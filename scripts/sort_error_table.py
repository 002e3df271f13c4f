"""The paper's Table 1 on the B200 path: per sort mode, the
sort error delta (metrics.py:46-73, per-pixel maps accumulated by K6 during
the blend) and the render time relative to GlobalZ, on full C3 orbit views
and C5 yaw-sweep views (1080p).  Modes: GlobalZ (the 3DGS order),
Hierarchical 64/8/4, Window 4 / 8 / 16 / 24 and FullPerPixel (the exact
per-pixel order, delta = 0).  Times are per-stage CUDA events (one view at a
time, after a warm-up view) of the plain render (no sort-error map: the
instrumented K6 computes t on every blend, which GlobalZ otherwise skips).
usage: python scripts/sort_error_table.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_00525_b200 import (FullPerPixel, GlobalZ, Hierarchical, RenderConfig,  # noqa: E402
                                   Window, scenes)
from paper_2402_00525_b200.renderer import Renderer  # noqa: E402

MODES = [GlobalZ(), Hierarchical(), Window(4), Window(8), Window(16), Window(24), FullPerPixel()]
rows = []
for cfgname, views in (("C3", (0, 64, 128, 192)), ("C5", (0, 120))):
    sc, cams = scenes.config_scene(cfgname)
    for mode in MODES:
        r = Renderer(sc, mode, RenderConfig())
        cam0 = cams[views[0]]
        outs = r.alloc_outputs(cam0.width, cam0.height, sort_error=True)
        plain = r.alloc_outputs(cam0.width, cam0.height)   # timing: the plain render
        r.render_into(cam0, plain, stats=True, timings=True)         # warm-up
        for v in views:
            r.render_into(cams[v], outs, stats=True)                 # delta map (XM_SERR)
            pp = outs["sort_error"].double().cpu().numpy()
            st = r.render_into(cams[v], plain, stats=True, timings=True)
            rows.append({"config": cfgname, "view": v, "mode": type(mode).__name__ +
                         (f"({mode.size})" if isinstance(mode, Window) else ""),
                         "delta_max": float(pp.max()), "delta_avg": float(pp.mean()),
                         "frac_pixels_nonzero": float((pp > 0).mean()),
                         "entries": int(st.bin_entries),
                         "ms_render": float(st.ms_blend),
                         "ms_view": float(st.ms_project + st.ms_duplicate + st.ms_sort +
                                          st.ms_blend)})
            print(json.dumps(rows[-1]), flush=True)
        del r, outs, plain
summ = {}
for r_ in rows:
    summ.setdefault((r_["config"], r_["mode"]), []).append(r_)
table = {}
for (c, m), v in summ.items():
    gz = summ[(c, "GlobalZ")]
    table[f"{c} {m}"] = {
        "delta_max": max(x["delta_max"] for x in v),
        "delta_avg": float(np.mean([x["delta_avg"] for x in v])),
        "ms_render": float(np.mean([x["ms_render"] for x in v])),
        "ms_view": float(np.mean([x["ms_view"] for x in v])),
        "render_vs_globalz": float(np.mean([x["ms_render"] for x in v]) /
                                   np.mean([x["ms_render"] for x in gz])),
        "view_vs_globalz": float(np.mean([x["ms_view"] for x in v]) /
                                 np.mean([x["ms_view"] for x in gz])),
        "views": len(v)}
print(json.dumps(table, indent=1))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump({"per_view": rows, "summary": table}, f, indent=1)
