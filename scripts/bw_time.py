"""Backward-pass timing on a full C3 view (Hierarchical): stp_backward =
K1-K5 + two K6 replays; device time by CUDA events around the call."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_00525_b200 import Hierarchical, GlobalZ, RenderConfig, scenes
from paper_2402_00525_b200.renderer import Renderer
sc, cams = scenes.config_scene("C3", n_views=8)
res = {}
for mode in (Hierarchical(), GlobalZ()):
    r = Renderer(sc, mode, RenderConfig())
    cam = cams[0]
    up = torch.randn((cam.height, cam.width, 3), dtype=torch.float64, device="cuda")
    r.backward(cam, up)   # warm (sizes the workspace)
    outs = r.alloc_outputs(cam.width, cam.height)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); e0.record()
        g = r.backward(cam, up)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    fw = []
    for _ in range(5):
        torch.cuda.synchronize(); e0.record()
        r.render_into(cam, outs)
        e1.record(); torch.cuda.synchronize(); fw.append(e0.elapsed_time(e1))
    res[type(mode).__name__] = {"backward_ms_incl_host": float(np.median(ts)),
                                "forward_ms": float(np.median(fw)), "kept": int(len(g.d_opacity))}
print(json.dumps(res))
