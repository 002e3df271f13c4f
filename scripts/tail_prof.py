"""K6 load-balance tail: per-warp start/end times of the persistent render
kernel (needs a -DSTP_TAIL_PROF build; instrumented, never a bench number)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_00525_b200 import scenes, Hierarchical, RenderConfig
from paper_2402_00525_b200.renderer import Renderer

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C3"
sc, cams = scenes.config_scene(cfgname, n_views=8)
r = Renderer(sc, Hierarchical(), RenderConfig())
res = []
for v in (0, 5):
    cam = cams[v]
    outs = r.alloc_outputs(cam.width, cam.height)
    for _ in range(2):
        st = r.render_into(cam, outs, stats=True, timings=True)
    L = r.ws.layout(r.scene.n, cam.width, cam.height)
    base = 336 + 256 * 64 + 256 * 4
    c = r.ws.buf[L.counters: L.counters + (base + 8192) * 8].view(torch.int64).cpu().numpy()
    se = c[base: base + 8192].reshape(4096, 2)
    se = se[se[:, 1] > 0].astype(np.float64)
    t0 = se[:, 0].min()
    s, e = (se[:, 0] - t0) / 1e3, (se[:, 1] - t0) / 1e3   # us
    q = np.percentile(e, [0, 10, 50, 90, 99, 100])
    busy = (e - s).sum() / (len(e) * e.max())
    res.append({"view": v, "K6_ms": st.ms_blend, "warps": int(len(e)),
                "start_us_max": round(float(s.max()), 1),
                "end_us_pct[0,10,50,90,99,100]": [round(float(x), 1) for x in q],
                "warp_busy_frac": round(float(busy), 4)})
print(json.dumps(res, indent=1))
