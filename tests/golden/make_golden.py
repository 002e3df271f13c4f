"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Each fixture stores float32 scene inputs (the reference is fed exactly these
values, widened to float64), the camera, the mode/config, and the reference's
outputs: projection stats and SplatBatch, the sorted tile lists
(``bin_and_sort``), the frame (colour / transmittance / depth) and per-pixel
blend records.  The files are committed; nothing on the GPU box reads
/root/reference.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("SPLATSORT_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import splatsort as S  # noqa: E402
from splatsort.fixtures import random_cloud  # noqa: E402

from paper_2402_00525_b200 import scenes  # noqa: E402


def to_gaussians(arrs):
    n = len(arrs["opacity"])
    sh = np.zeros((n, 16, 3))
    k = arrs["sh"].shape[1]
    sh[:, :k] = arrs["sh"]
    return [S.Gaussian3D(mean=arrs["means"][i].astype(np.float64),
                         rotation=arrs["quats"][i].astype(np.float64),
                         scale=arrs["scales"][i].astype(np.float64),
                         opacity=float(arrs["opacity"][i]), sh=sh[i]) for i in range(n)]


def from_gaussians(gs):
    if not gs:
        return {"means": np.zeros((0, 3), np.float32), "quats": np.zeros((0, 4), np.float32),
                "scales": np.zeros((0, 3), np.float32), "opacity": np.zeros(0, np.float32),
                "sh": np.zeros((0, 16, 3), np.float32)}
    return scenes.to_f32_scene({
        "means": np.stack([g.mean for g in gs]), "quats": np.stack([g.rotation for g in gs]),
        "scales": np.stack([g.scale for g in gs]), "opacity": np.array([g.opacity for g in gs]),
        "sh": np.stack([g.sh for g in gs])})


def ball(mean, scale, opacity, rgb, rot=(1, 0, 0, 0)):
    sh = np.zeros((16, 3))
    sh[0] = (np.asarray(rgb, dtype=np.float64) - 0.5) / 0.28209479177387814
    return S.Gaussian3D(mean=mean, rotation=rot, scale=[scale] * 3 if np.isscalar(scale) else scale,
                        opacity=opacity, sh=sh)


def axis_cam(w, h, f=110.0, R=None, pos=None, cx=None, cy=None):
    return S.Camera(rotation=np.eye(3) if R is None else R,
                    position=np.zeros(3) if pos is None else pos,
                    fx=f, fy=f, width=w, height=h, cx=cx, cy=cy)


def save(name, arrs, cam, mode, cfg, sh_coeffs=16, rec_pixels=None, store_batch=True):
    arrs = dict(arrs)
    arrs["sh"] = np.ascontiguousarray(arrs["sh"][:, :sh_coeffs])
    gs = to_gaussians(arrs)
    cfg_d = dict(tile_size=cfg.tile_size, opacity_eps=cfg.opacity_eps,
                 termination=cfg.termination, alpha_cap=cfg.alpha_cap,
                 background=[float(v) for v in cfg.background], near=cfg.near,
                 guard_band=cfg.guard_band, dilation=cfg.dilation,
                 inv_scale_clamp=cfg.inv_scale_clamp, with_depth=cfg.with_depth,
                 exact_tile_culling=cfg.exact_tile_culling)
    if isinstance(mode, S.GlobalZ):
        mode_d = dict(mode="globalz")
    elif isinstance(mode, S.FullPerPixel):
        mode_d = dict(mode="full")
    elif isinstance(mode, S.Window):
        mode_d = dict(mode="window", size=mode.size)
    else:
        mode_d = dict(queue_tail=mode.queue_tail, queue_mid=mode.queue_mid,
                      queue_head=mode.queue_head, batch_load=mode.batch_load,
                      batch_mid=mode.batch_mid, batch_head=mode.batch_head,
                      mid_depth_at_center=mode.mid_depth_at_center)
    cfg_rec = S.RenderConfig(**{**cfg_d, "capture_records": True})
    t0 = time.time()
    frame = S.render(gs, cam, mode, cfg_rec)
    dt = time.time() - t0
    batch, pstats = S.project_scene(gs, cam, near=cfg.near, guard=cfg.guard_band,
                                    dilation=cfg.dilation, inv_scale_clamp=cfg.inv_scale_clamp,
                                    eps=cfg.opacity_eps)
    bins = S.bin_and_sort(batch, cam, mode, cfg)
    gw = -(-cam.width // cfg.tile_size)
    tile_id = np.concatenate([np.full(len(b), b.tile_y * gw + b.tile_x, np.int32) for b in bins]) \
        if bins else np.zeros(0, np.int32)
    splat = np.concatenate([b.splat for b in bins]).astype(np.int32) if bins else np.zeros(0, np.int32)
    key = np.concatenate([b.key for b in bins]) if bins else np.zeros(0)
    H, W = cam.height, cam.width
    if rec_pixels is None:
        ys, xs = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        rec_pixels = np.stack([ys.ravel(), xs.ravel()], 1)
    rec_pixels = np.asarray(rec_pixels, dtype=np.int32)
    counts = np.array([len(frame.records[y][x]) for y, x in rec_pixels], dtype=np.int32)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    rs = np.zeros(int(offs[-1]), np.int32)
    rt = np.zeros(int(offs[-1]), np.float32)
    ra = np.zeros(int(offs[-1]), np.float32)
    for i, (y, x) in enumerate(rec_pixels):
        r = frame.records[y][x]
        rs[offs[i]:offs[i + 1]] = r.splat
        rt[offs[i]:offs[i + 1]] = r.depth
        ra[offs[i]:offs[i + 1]] = r.alpha
    out = dict(
        means=arrs["means"], quats=arrs["quats"], scales=arrs["scales"],
        opacity=arrs["opacity"], sh=arrs["sh"],
        cam_R=cam.rotation, cam_pos=cam.position,
        cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
        cam_size=np.array([cam.width, cam.height], np.int32),
        cfg_json=np.array(json.dumps(cfg_d)), mode_json=np.array(json.dumps(mode_d)),
        proj_stats=np.array([pstats[k] for k in ("input", "behind", "guard", "degenerate", "kept")]),
        source_index=batch.source_index.astype(np.int32),
        bin_tile=tile_id, bin_splat=splat,
        color=frame.color.astype(np.float32), transmittance=frame.transmittance.astype(np.float32),
        color64_absmax=np.array(np.abs(frame.color).max() if frame.color.size else 0.0),
        rec_pixels=rec_pixels, rec_offsets=offs, rec_splat=rs, rec_t=rt, rec_alpha=ra,
        ref_seconds=np.array(dt),
    )
    if cfg.with_depth:
        out["depth"] = frame.depth.astype(np.float32)
    if store_batch:
        out.update(b_mean2d=batch.mean2d, b_conic=batch.conic, b_color=batch.color,
                   b_radius=batch.radius, b_inv_cov3=batch.inv_cov3,
                   b_inv_cov_center=batch.inv_cov_center, bin_key=key)
        if isinstance(mode, S.GlobalZ):
            out.update(b_global_depth=batch.global_depth, b_center_dist=batch.center_dist)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: kept={pstats['kept']} entries={len(splat)} tiles={len(bins)} "
          f"ref={dt:.2f}s -> {os.path.getsize(path) / 1e6:.2f} MB", flush=True)


def main(only=None, only_grads=None):
    H = S.Hierarchical()
    jobs = {}

    # 1. dense random cloud (reference fixture), background + depth
    def cloud300():
        gs, cams, _ = random_cloud(300, seed=5)
        save("cloud300", from_gaussians(gs), cams[0], H,
             S.RenderConfig(with_depth=True, background=np.array([0.1, 0.2, 0.3])))
    jobs["cloud300"] = cloud300

    # 2. rotated camera of the same fixture (3 deg yaw), SH degree 3
    def cloud300_rot():
        gs, cams, _ = random_cloud(300, seed=6)
        save("cloud300_rot", from_gaussians(gs), cams[1], H, S.RenderConfig(with_depth=True))
    jobs["cloud300_rot"] = cloud300_rot

    # 3. shallow scene: <= 4 contributions per ray (test_rasterizer.py:398-412)
    def shallow():
        gs = [ball([0.0, 0.0, 2.0], 0.25, 0.6, [0.8, 0.2, 0.2]),
              ball([0.05, 0.02, 2.5], 0.25, 0.6, [0.2, 0.8, 0.2]),
              ball([-0.04, 0.03, 3.1], 0.25, 0.6, [0.2, 0.2, 0.8]),
              ball([0.02, -0.05, 3.7], 0.25, 0.6, [0.7, 0.7, 0.1])]
        save("shallow", from_gaussians(gs), axis_cam(48, 48), H, S.RenderConfig(with_depth=True))
    jobs["shallow"] = shallow

    # 4. edge cases: coincident pair (rank tie-break), near/guard/low-opacity culls
    def edges():
        gs = [ball([0.0, 0.0, 2.0], 0.1, 0.5, [1.0, 0.0, 0.0]),
              ball([0.0, 0.0, 2.0], 0.1, 0.5, [0.0, 0.0, 1.0]),
              ball([0.3, 0.1, 0.1], 0.1, 0.5, [0.0, 1.0, 0.0]),      # behind near plane
              ball([5.0, 0.0, 2.0], 0.1, 0.5, [0.0, 1.0, 0.0]),      # outside guard band
              ball([-0.2, 0.2, 2.0], 0.2, 1e-4, [1.0, 1.0, 0.0]),    # below eps
              ball([0.2, -0.2, 2.5], 0.3, 1.0, [1.0, 1.0, 1.0]),     # alpha cap
              ball([-0.3, -0.3, 3.0], [0.6, 0.01, 0.01], 0.9, [0.3, 0.6, 0.9],
                   rot=[0.9238795, 0.0, 0.0, 0.3826834])]           # elongated, rotated
        save("edges", from_gaussians(gs), axis_cam(37, 29, f=40.0), H,
             S.RenderConfig(with_depth=True, background=np.array([0.5, 0.5, 0.5])))
    jobs["edges"] = edges

    # 5. SH degree 3 frustum cloud, rotated + translated camera, off-centre
    #    principal point, ragged image size (partial tiles and sub-tiles)
    def sh3_border():
        arrs = scenes.frustum_cloud(1500, 21, 203, 117, 150.0, z_lo=1.0, z_hi=5.0)
        arrs["scales"] = arrs["scales"] * 4.0
        pos = np.array([0.1, -0.05, -0.2])
        R = scenes.look_at(pos, np.array([0.15, 0.0, 3.0]))
        cam = axis_cam(203, 117, f=150.0, R=R, pos=pos, cx=97.3, cy=61.9)
        save("sh3_border", scenes.to_f32_scene(arrs), cam, H, S.RenderConfig(with_depth=True))
    jobs["sh3_border"] = sh3_border

    # 6. mode variants: mid_depth_at_center, non-default queues, coarse binning
    def variants():
        gs, cams, _ = random_cloud(200, seed=11)
        a = from_gaussians(gs)
        save("var_center", a, cams[0], S.Hierarchical(mid_depth_at_center=True),
             S.RenderConfig(with_depth=True))
        save("var_queues", a, cams[0], S.Hierarchical(queue_tail=96, queue_mid=12, queue_head=8),
             S.RenderConfig(with_depth=True))
        save("var_coarse", a, cams[0], H,
             S.RenderConfig(with_depth=True, exact_tile_culling=False))
        save("var_q4", a, cams[0], S.Hierarchical(queue_mid=4, queue_head=1),
             S.RenderConfig(with_depth=True))
    jobs["variants"] = variants

    # 7. empty scene -> background
    def empty():
        save("empty", from_gaussians([]), axis_cam(32, 32), H,
             S.RenderConfig(background=np.array([0.2, 0.4, 0.6])))
    jobs["empty"] = empty

    # 8. config #1 (BASELINE.json configs[0]): 10k random Gaussians, SH0, 256^2
    def c1():
        sc, cams = scenes.config_scene("C1")
        rng = np.random.default_rng(123)
        pix = np.stack([rng.integers(0, 256, 400), rng.integers(0, 256, 400)], 1)
        save("c1", sc, cams[0], H, S.RenderConfig(with_depth=True), sh_coeffs=1,
             rec_pixels=pix, store_batch=False)
    jobs["c1"] = c1

    # 9. GlobalZ (the 3DGS baseline order: one view-z key per splat, coarse
    #    bins by default) on the same scenes, plus GlobalZ with exact culling
    def globalz():
        G = S.GlobalZ()
        gs, cams, _ = random_cloud(300, seed=5)
        save("gz_cloud300", from_gaussians(gs), cams[0], G,
             S.RenderConfig(with_depth=True, background=np.array([0.1, 0.2, 0.3])))
        arrs = scenes.frustum_cloud(1500, 21, 203, 117, 150.0, z_lo=1.0, z_hi=5.0)
        arrs["scales"] = arrs["scales"] * 4.0
        pos = np.array([0.1, -0.05, -0.2])
        R = scenes.look_at(pos, np.array([0.15, 0.0, 3.0]))
        cam = axis_cam(203, 117, f=150.0, R=R, pos=pos, cx=97.3, cy=61.9)
        save("gz_sh3_border", scenes.to_f32_scene(arrs), cam, G, S.RenderConfig(with_depth=True))
        gs, cams, _ = random_cloud(200, seed=11)
        save("gz_exact", from_gaussians(gs), cams[0], G,
             S.RenderConfig(with_depth=True, exact_tile_culling=True))
    jobs["globalz"] = globalz

    # 10. FullPerPixel (the exact per-ray order) and Window(k) (per-pixel
    #     resorting window over the per-tile-depth stream)
    def pixelsort():
        gs, cams, _ = random_cloud(300, seed=5)
        a = from_gaussians(gs)
        save("full_cloud300", a, cams[0], S.FullPerPixel(),
             S.RenderConfig(with_depth=True, background=np.array([0.1, 0.2, 0.3])))
        save("win8_cloud300", a, cams[0], S.Window(8), S.RenderConfig(with_depth=True))
        save("win2_cloud300", a, cams[0], S.Window(2), S.RenderConfig(with_depth=True))
        arrs = scenes.frustum_cloud(1500, 21, 203, 117, 150.0, z_lo=1.0, z_hi=5.0)
        arrs["scales"] = arrs["scales"] * 4.0
        pos = np.array([0.1, -0.05, -0.2])
        R = scenes.look_at(pos, np.array([0.15, 0.0, 3.0]))
        cam = axis_cam(203, 117, f=150.0, R=R, pos=pos, cx=97.3, cy=61.9)
        save("full_sh3_border", scenes.to_f32_scene(arrs), cam, S.FullPerPixel(),
             S.RenderConfig(with_depth=True))
        save("win8_sh3_border", scenes.to_f32_scene(arrs), cam, S.Window(8),
             S.RenderConfig(with_depth=True))
    jobs["pixelsort"] = pixelsort

    # 10b. Window(k) beyond the register window (k > 16): the paper's Table-1
    #      window 24 and a 64-entry window whose overflow
    #      path still triggers on the deep border fixture
    def windows():
        gs, cams, _ = random_cloud(300, seed=5)
        a = from_gaussians(gs)
        save("win24_cloud300", a, cams[0], S.Window(24), S.RenderConfig(with_depth=True))
        arrs = scenes.frustum_cloud(1500, 21, 203, 117, 150.0, z_lo=1.0, z_hi=5.0)
        arrs["scales"] = arrs["scales"] * 4.0
        pos = np.array([0.1, -0.05, -0.2])
        R = scenes.look_at(pos, np.array([0.15, 0.0, 3.0]))
        cam = axis_cam(203, 117, f=150.0, R=R, pos=pos, cx=97.3, cy=61.9)
        save("win64_sh3_border", scenes.to_f32_scene(arrs), cam, S.Window(64),
             S.RenderConfig(with_depth=True))
    jobs["windows"] = windows

    # 11. backward pass (gradients.py:84-162): reference gradients w.r.t. the
    #     projected batch for a seeded upstream dL/dcolour, per fixture/mode
    def grads():
        from splatsort import gradients as SG
        for fx in (only_grads or ("cloud300", "shallow", "sh3_border", "gz_cloud300",
                                  "win8_cloud300", "edges", "win24_cloud300")):
            z = np.load(os.path.join(HERE, f"{fx}.npz"))
            d = {k: z[k] for k in z.files}
            arrs = {k: d[k] for k in ("means", "quats", "scales", "opacity", "sh")}
            gs = to_gaussians(arrs)
            fxi, fyi, cxi, cyi = d["cam_intr"]
            w, h = (int(v) for v in d["cam_size"])
            cam = S.Camera(rotation=d["cam_R"], position=d["cam_pos"], fx=fxi, fy=fyi,
                           width=w, height=h, cx=cxi, cy=cyi)
            cfg = S.RenderConfig(**json.loads(str(d["cfg_json"])))
            md = json.loads(str(d["mode_json"]))
            kind = md.pop("mode", "hierarchical")
            mode = {"globalz": S.GlobalZ, "full": S.FullPerPixel}.get(kind)
            mode = mode() if mode else (S.Window(**md) if kind == "window" else S.Hierarchical(**md))
            batch, _ = S.project_scene(gs, cam, near=cfg.near, guard=cfg.guard_band,
                                       dilation=cfg.dilation,
                                       inv_scale_clamp=cfg.inv_scale_clamp, eps=cfg.opacity_eps)
            up = np.random.default_rng(99).normal(0, 1, (h, w, 3))
            g = SG.backward_render(batch, cam, mode, up, cfg)
            path = os.path.join(HERE, f"grad_{fx}.npz")
            np.savez_compressed(path, upstream=up, d_color=g.d_color, d_opacity=g.d_opacity,
                                d_mean2d=g.d_mean2d, d_conic=g.d_conic,
                                d_background=g.d_background)
            print(f"grad_{fx}: n={len(g.d_opacity)} -> {os.path.getsize(path) / 1e6:.2f} MB",
                  flush=True)
    jobs["grads"] = grads

    # 12. scene / camera I/O (scene_io.py:189-417): a 3DGS PLY checkpoint and a
    #     cameras.json written by the reference, plus what its loaders return
    def io():
        from splatsort import scene_io as SIO
        gs, cams, _ = random_cloud(200, seed=17)
        for g in gs:   # full SH so f_rest carries data
            g.sh[1:] = np.random.default_rng(len(g.sh)).normal(0, 0.2, (15, 3))
        ply = os.path.join(HERE, "io_cloud200.ply")
        SIO.save_ply(gs, ply)
        back = SIO.load_ply(ply)
        cj = os.path.join(HERE, "io_cams.json")
        SIO.save_cameras(cams, cj)
        cb = SIO.load_cameras(cj)
        np.savez_compressed(os.path.join(HERE, "io_expected.npz"),
                            means=np.stack([g.mean for g in back]),
                            quats=np.stack([g.rotation for g in back]),
                            scales=np.stack([g.scale for g in back]),
                            opacity=np.array([g.opacity for g in back]),
                            sh=np.stack([g.sh for g in back]),
                            cam_R=np.stack([c.rotation for c in cb]),
                            cam_pos=np.stack([c.position for c in cb]),
                            cam_intr=np.array([[c.fx, c.fy, c.cx, c.cy] for c in cb]),
                            cam_size=np.array([[c.width, c.height] for c in cb]))
        print(f"io: {len(back)} Gaussians, {len(cb)} cameras", flush=True)
    jobs["io"] = io

    # 13. view consistency (metrics.py:80-255): three depth frames of a small
    #     yaw sweep rendered by the reference, its analytic flows, warps,
    #     occlusion masks and the squared-error consistency score
    def consistency():
        from splatsort import metrics as SM
        arrs = scenes.frustum_cloud(2000, 31, 96, 72, 80.0, z_lo=2.0, z_hi=6.0)
        gs = to_gaussians(scenes.to_f32_scene(arrs))
        cams = []
        for k in range(3):
            a = np.deg2rad(1.5 * k)
            R = np.array([[np.cos(a), 0, -np.sin(a)], [0, 1, 0], [np.sin(a), 0, np.cos(a)]])
            cams.append(axis_cam(96, 72, f=80.0, R=R, pos=np.array([0.02 * k, 0.0, 0.0])))
        cfg = S.RenderConfig(with_depth=True)
        fr = [S.render(gs, c, S.Hierarchical(), cfg) for c in cams]
        out = {}
        for k, f in enumerate(fr):
            out[f"color{k}"], out[f"depth{k}"], out[f"tn{k}"] = f.color, f.depth, f.transmittance
            out[f"R{k}"], out[f"pos{k}"] = cams[k].rotation, cams[k].position
        fw, bw = {}, {}
        for i in range(3):
            for j in range(3):
                if i != j:
                    fl, va = SM.analytic_flow(fr[i], cams[i], cams[j])
                    out[f"flow{i}{j}"], out[f"valid{i}{j}"] = fl, va
                    (fw if j > i else bw)[(i, j)] = (fl, va)
        wa, wv = SM.warp_frame(fr[1].color, out["flow01"])
        out["warp01"], out["warpvalid01"] = wa, wv
        out["occ01"] = SM.occlusion_mask(out["flow01"], out["flow10"])
        rep = SM.view_consistency(fr, fw, bw, offsets=(1, 2), metric="both", crop=4)
        out["mse_t"] = np.array([rep.mse_t[1], rep.mse_t[2]])
        out["flip_t"] = np.array([rep.flip_t[1], rep.flip_t[2]])
        from splatsort.flip import flip_error_map
        out["flip01"] = flip_error_map(fr[0].color, wa)
        np.savez_compressed(os.path.join(HERE, "io_consistency.npz"), **out)
        print("consistency:", rep.mse_t, flush=True)
    jobs["consistency"] = consistency

    for name, fn in jobs.items():
        if only and name not in only:
            continue
        fn()


if __name__ == "__main__":
    # make_golden.py [job ...] [--grads fixture ...]
    argv = sys.argv[1:]
    grads_only = None
    if "--grads" in argv:
        i = argv.index("--grads")
        grads_only, argv = tuple(argv[i + 1:]), argv[:i]
    main(argv or None, grads_only)
