"""The UNMODIFIED reference (baseline/_ref, splatsort) as a CPU point on the
benchmark's workload, by the protocol of SURVEY.md §8(d): on one C3 view
(3M Gaussians, 1080p, Hierarchical 64/8/4), time `project_scene` and
`bin_and_sort` in full, then the reference's own per-tile seam
`hierarchy.render_tile(_TileCtx(...), tbin, mode)` (rasterizer.py:645-655)
on a seeded stratified sample of tiles, and extrapolate the render stage by
the frame's total bin entries at the sample's per-entry rate.  One worker
(the reference's tile pool is GIL-bound: w = 1 is its fastest setting,
SURVEY.md §6).  Writes a JSON that bench.py attaches to cpu_baseline.

usage: python scripts/reference_cpu_point.py OUT.json [config] [view] [tiles]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(1, ROOT)
import numpy as np  # noqa: E402

import splatsort as S  # noqa: E402
from splatsort import hierarchy  # noqa: E402
from splatsort.rasterizer import _TileCtx  # noqa: E402

from paper_2402_00525_b200 import scenes  # noqa: E402  (the synthetic scene generator)

out_path = sys.argv[1]
cfgname = sys.argv[2] if len(sys.argv) > 2 else "C3"
view = int(sys.argv[3]) if len(sys.argv) > 3 else 5
n_tiles = int(sys.argv[4]) if len(sys.argv) > 4 else 48


class G:
    """Duck-typed Gaussian3D (gaussian_math.py:353-357 reads these five
    attributes); avoids 3M dataclass __post_init__ copies."""
    __slots__ = ("mean", "rotation", "scale", "opacity", "sh")

    def __init__(self, m, q, s, o, sh):
        self.mean, self.rotation, self.scale, self.opacity, self.sh = m, q, s, o, sh


t0 = time.perf_counter()
sc, cams = scenes.config_scene(cfgname)
cam0 = cams[view]
cam = S.Camera(rotation=np.asarray(cam0.rotation, dtype=np.float64),
               position=np.asarray(cam0.position, dtype=np.float64), fx=cam0.fx, fy=cam0.fy,
               width=cam0.width, height=cam0.height, cx=cam0.cx, cy=cam0.cy)
m = sc["means"].astype(np.float64)
q = sc["quats"].astype(np.float64)
s = sc["scales"].astype(np.float64)
o = sc["opacity"].astype(np.float64)
sh = np.zeros((len(o), 16, 3))
sh[:, : sc["sh"].shape[1]] = sc["sh"]
gs = [G(m[i], q[i], s[i], float(o[i]), sh[i]) for i in range(len(o))]
t_setup = time.perf_counter() - t0
mode, cfg = S.Hierarchical(), S.RenderConfig(workers=1)

t0 = time.perf_counter()
batch, pstats = S.project_scene(gs, cam, near=cfg.near, guard=cfg.guard_band,
                                dilation=cfg.dilation, inv_scale_clamp=cfg.inv_scale_clamp,
                                eps=cfg.opacity_eps)
t_project = time.perf_counter() - t0
del gs
t0 = time.perf_counter()
bins = S.bin_and_sort(batch, cam, mode, cfg, timings={})
t_bin = time.perf_counter() - t0
E = int(sum(len(b) for b in bins))

# stratified seeded sample: tiles ranked by entry count, one per stratum
rng = np.random.default_rng(0)
order = np.argsort([len(b) for b in bins], kind="stable")
strata = np.array_split(order, n_tiles)
pick = [int(st[rng.integers(len(st))]) for st in strata if len(st)]
t_tiles, e_tiles = 0.0, 0
for i in pick:
    tb = bins[i]
    t0 = time.perf_counter()
    hierarchy.render_tile(_TileCtx(batch, cam, cfg, tb.tile_x, tb.tile_y), tb, mode)
    t_tiles += time.perf_counter() - t0
    e_tiles += len(tb)
rate = t_tiles / max(e_tiles, 1)
t_render = rate * E
total = t_project + t_bin + t_render
res = {"config": cfgname, "view": view, "mode": "hierarchical:64/8/4", "workers": 1,
       "gaussians": int(len(o)), "kept": int(pstats["kept"]), "bin_entries": E,
       "tiles": len(bins), "tiles_sampled": len(pick), "entries_sampled": e_tiles,
       "s_project_scene": t_project, "s_bin_and_sort": t_bin,
       "s_render_sampled": t_tiles, "s_per_entry": rate, "s_render_extrapolated": t_render,
       "s_per_view": total, "views_per_s": 1.0 / total, "s_setup_not_timed": t_setup,
       "host_threads_available": len(os.sched_getaffinity(0)),
       "numpy": np.__version__, "reference": os.path.dirname(S.__file__)}
print(json.dumps(res, indent=1))
with open(out_path, "w") as f:
    json.dump(res, f, indent=1)
