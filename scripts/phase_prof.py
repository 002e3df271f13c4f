"""Per-phase warp-cycle breakdown of K6 (needs a -DSTP_PHASE_PROF build)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_00525_b200 import scenes, Hierarchical, RenderConfig
from paper_2402_00525_b200.renderer import Renderer

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C3"
sc, cams = scenes.config_scene(cfgname, n_views=8)
r = Renderer(sc, Hierarchical(), RenderConfig())
cam = cams[0]
outs = r.alloc_outputs(cam.width, cam.height)
for _ in range(2):
    st = r.render_into(cam, outs, stats=True, timings=True)
L = r.ws.layout(r.scene.n, cam.width, cam.height)
c = r.ws.buf[L.counters: L.counters + 80 * 8].view(torch.int64).cpu().numpy()
prof = c[32:38].astype(np.float64)
names = ["load(+cull+d4)", "sort+merge", "push_mid", "pixel", "item_epilogue", "item_prologue"]
tot = prof.sum()
stat = c[48:80].astype(np.int64)
snames = ["load_evals(entry,subtile)", "kept_4x4", "batches", "batches_nonempty",
          "pixel_slots(lane,entry)", "pixel_evals(T>=term)", "alpha_pass", "evals_in_all_fail_quads", "pixel_warp_steps", "consume_calls", "mid_merges", "mid_merges_steady",
          "compact_halves_nk_gt1", "compact_halves_sorted", "tail_merges", "tail_merges_append",
          "head_push_full(lanes)", "head_push_full_after_all(lanes)", "head_push_full(warp_steps)",
          "head_push_full_all_after(warp_steps)", "mid_steady_append(quad_merges)",
          "mid_steady_all_quads_append(warp_merges)"]
print(json.dumps({"K6_ms": st.ms_blend, "entries": int(st.bin_entries),
                  "stats": {n: int(v) for n, v in zip(snames, stat)},
                  "phase_frac": {n: round(float(v / tot), 4) for n, v in zip(names, prof)},
                  "warp_cycles_G": round(tot / 1e9, 3)}))
