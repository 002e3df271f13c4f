"""Sort error at scale (the paper's Table 1 delta, metrics.py:46-73) on full
C3 / C5 views, GlobalZ vs Hierarchical, from the GPU's per-pixel maps.
usage: python scripts/sort_error_table.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_00525_b200 import GlobalZ, Hierarchical, RenderConfig, scenes  # noqa: E402
from paper_2402_00525_b200.renderer import Renderer  # noqa: E402

rows = []
for cfgname, views in (("C3", (0, 64, 128, 192)), ("C5", (0, 8))):
    sc, cams = scenes.config_scene(cfgname, n_views=256 if cfgname == "C3" else 16)
    for mode in (GlobalZ(), Hierarchical()):
        r = Renderer(sc, mode, RenderConfig())
        for v in views:
            out = r.frame(cams[v], sort_error=True)
            pp = out.sort_error
            rows.append({"config": cfgname, "view": v, "mode": out.stats["mode"],
                         "delta_max": float(pp.max()), "delta_avg": float(pp.mean()),
                         "frac_pixels_nonzero": float((pp > 0).mean()),
                         "entries": out.stats["bin_entries"]})
            print(json.dumps(rows[-1]), flush=True)
summ = {}
for r_ in rows:
    k = f'{r_["config"]} {r_["mode"]}'
    summ.setdefault(k, []).append(r_)
table = {k: {"delta_max": max(x["delta_max"] for x in v),
             "delta_avg": float(np.mean([x["delta_avg"] for x in v])),
             "views": len(v)} for k, v in summ.items()}
print(json.dumps(table, indent=1))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump({"per_view": rows, "summary": table}, f, indent=1)
