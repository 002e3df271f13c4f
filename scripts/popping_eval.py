"""Popping / view consistency at scale (the paper's temporal-consistency
evaluation; metrics.view_consistency on the C5 sweep): N consecutive 1080p
frames of the C5 yaw sweep rendered on the GPU under GlobalZ, Hierarchical and
FullPerPixel, analytic flows from the rendered depth, FLIP and squared-error
consistency at frame offsets 1 and 7, all on the device.
usage: python scripts/popping_eval.py [n_frames] [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_00525_b200 import FullPerPixel, GlobalZ, Hierarchical, RenderConfig, scenes  # noqa: E402
from paper_2402_00525_b200 import consistency as C  # noqa: E402
from paper_2402_00525_b200.renderer import Renderer  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 16
sc, cams = scenes.config_scene("C5")
cams = cams[100:100 + nf]
dev = torch.device("cuda")
res = {"config": "C5 (1.5M half-density garden, 1080p), frames 100..%d of the 240-frame "
                 "30-degree yaw sweep" % (100 + nf - 1), "frames": nf}
for mode in (GlobalZ(), Hierarchical(), FullPerPixel()):
    t0 = time.time()
    r = Renderer(sc, mode, RenderConfig(with_depth=True))
    fr = [r.frame(c, device_output=True) for c in cams]
    fw = {(i, j): C.analytic_flow(fr[i], cams[i], cams[j], device=dev)
          for i in range(nf) for j in range(i + 1, nf) if j - i in (1, 7)}
    bw = {(j, i): C.analytic_flow(fr[j], cams[j], cams[i], device=dev)
          for i in range(nf) for j in range(i + 1, nf) if j - i in (1, 7)}
    rep = C.view_consistency(fr, fw, bw, offsets=(1, 7), metric="both", device=dev)
    name = type(mode).__name__
    res[name] = {"flip_t": rep.flip_t, "mse_t": rep.mse_t, "seconds": round(time.time() - t0, 1)}
    print(name, json.dumps(res[name]), flush=True)
if len(sys.argv) > 2:
    with open(sys.argv[2], "w") as f:
        json.dump(res, f, indent=1)
