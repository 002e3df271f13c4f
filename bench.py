#!/usr/bin/env python
"""Benchmark: hierarchical-sorted Gaussian splatting views/sec on B200.

Workload (BASELINE.json configs[2], the metric's "1080p, 3M Gaussians"):
C3 = synthetic 3M-Gaussian garden-scale scene (SH degree 3), a 256-view
1080p orbit.  One step = one full view per GPU through the C ABI (K0..K6:
preprocess, scan, duplicate, onesweep sort, ranges, hierarchical render).
Views are sharded across ranks with no collective on the hot path (weak
scaling: each rank renders one view per step); the scene is replicated once
by an NCCL broadcast from rank 0.

    python bench.py [--gpus N --steps K --warmup W]           # this framework
    python bench.py --impl reference [...]                     # CPU oracle arm

Prints ONE JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("frames/sec at 1080p, 3M Gaussians (1 GPU); views/sec at 1/2/4/8 B200; HBM GB/s")
UNIT = "views/s"
WORKLOADS = {
    "C1": "C1: synthetic 10k random Gaussians (SH0), single 256x256 view",
    "C2": "C2: synthetic 1M Gaussians (SH3), single 1920x1080 view",
    "C3": "C3: synthetic 3M-Gaussian garden-scale scene (SH3), 256-view 1920x1080 orbit",
    "C4": "C4: synthetic 6M Gaussians (SH3) at 3840x2160, culling / queue stress",
    "C5": "C5: synthetic 1.5M half-density scene (SH3), 1080p rotation sweep",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=128)
    p.add_argument("--warmup", type=int, default=8)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="C3")
    p.add_argument("--mode", default="hierarchical",
                   help="sort mode: hierarchical (the paper's pipeline, default) or globalz "
                        "(the 3DGS baseline order, for the paper's A/B)")
    p.add_argument("--gaussians", type=int, default=None, help="override N (debug)")
    p.add_argument("--views", type=int, default=256)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--fast32", action="store_true",
                   help="K6 via the fp32-state certified kernel (A/B against the float64 one)")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--streams", type=int, default=2,
                   help="views in flight per GPU (one workspace + stream each): the next "
                        "view's preprocess/sort fills the SMs the previous view's render "
                        "kernel releases at its tail")
    p.add_argument("--cpu-seconds", type=float, default=120.0,
                   help="wall budget of the reference arm's timed steps")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1", "0x1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def b_alg(n, sh_k, n_v, e, p, with_depth=False):
    """SURVEY.md 8(d) algorithmic bytes of one view and of the K6 launch."""
    out_px = 20 if with_depth else 16
    view = n * 4 * (11 + 3 * sh_k) + 2 * 80 * n_v + 48 * e + out_px * p
    k6 = 80 * n_v + 12 * e + out_px * p
    return view, k6


# ----------------------------------------------------------------------------
# reference arm: the reference's algorithm on the host cores (oracle port)

def cpu_view_rate(scene, cams, views, budget_s, threads, mode=None):
    """Full views (project + bin_and_sort + render of every tile under the
    sort mode, hierarchical by default) of the C++ restatement of the
    reference, all host threads."""
    import oracle
    from paper_2402_00525_b200 import Hierarchical, RenderConfig
    mode = mode if mode is not None else Hierarchical()
    times = []
    t_all = time.perf_counter()
    for v in views:
        t0 = time.perf_counter()
        oracle.render(scene, cams[v], RenderConfig(), mode, threads=threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s:
            break
    return len(times) / sum(times), len(times), times


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2402_00525_b200 import scenes
    scene, cams = scenes.config_scene(args.config, n=args.gaussians, n_views=args.views)
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    from paper_2402_00525_b200.types import mode_name, parse_mode
    mode = parse_mode(args.mode)
    # warmup (bounded: at most 2 views)
    cpu_view_rate(scene, cams, list(range(min(args.warmup, 2))), 1e9, threads, mode)
    views = [s % len(cams) for s in range(args.steps)]
    rate, done, times = cpu_view_rate(scene, cams, views, args.cpu_seconds, threads, mode)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": ws,
        "steps": done, "warmup": min(args.warmup, 2), "ms_per_step": 1e3 / rate,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOADS[args.config.upper()], "gaussians": len(scene["opacity"]),
                                        "width": cams[0].width, "height": cams[0].height,
                                        "views": len(cams), "mode": mode_name(mode)},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{done} full {args.config.upper()} views (project + bin_and_sort + "
                                   f"{mode_name(mode)} render of all tiles) by oracle/stp_oracle.cpp, "
                                   f"the float64 C++ restatement of the reference pinned to its "
                                   f"golden outputs; requested steps={args.steps}, timed within "
                                   f"{args.cpu_seconds:.0f} s"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2402_00525_b200 import Hierarchical, RenderConfig, _lib, scenes
    from paper_2402_00525_b200.renderer import GaussianScene, Renderer, make_camera, make_config
    from paper_2402_00525_b200.types import mode_name, parse_mode

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # scene: generated on rank 0, replicated by NCCL broadcast (no hot-path collective)
    t_gen = time.perf_counter()
    if rank == 0:
        host_scene, cams = scenes.config_scene(args.config, n=args.gaussians, n_views=args.views)
        shapes = [list(host_scene[k].shape) for k in ("means", "quats", "scales", "opacity", "sh")]
    else:
        host_scene = None
        cams = scenes.config_cameras(args.config, n_views=args.views)
        shapes = None
    if world > 1:
        obj = [shapes]
        dist.broadcast_object_list(obj, src=0)
        shapes = obj[0]
    keys = ("means", "quats", "scales", "opacity", "sh")
    dev_t = {}
    for k, shp in zip(keys, shapes):
        if rank == 0:
            dev_t[k] = torch.from_numpy(host_scene[k]).to(dev)
        else:
            dev_t[k] = torch.empty(shp, dtype=torch.float32, device=dev)
        if world > 1:
            dist.broadcast(dev_t[k], src=0)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    gs = GaussianScene(dev_t["means"], dev_t["quats"], dev_t["scales"], dev_t["opacity"],
                       dev_t["sh"], dev)
    mode, cfg = parse_mode(args.mode), RenderConfig()
    r = Renderer(gs, mode, cfg, dev, fast32=args.fast32)
    lib = _lib.load()
    W, H = cams[0].width, cams[0].height
    n_views = len(cams)
    steps, warm = args.steps, args.warmup
    my_views = [((s * world + rank) % n_views) for s in range(warm + steps)]

    # size the workspace and collect per-view stats (also warms every view)
    outs = r.alloc_outputs(W, H)
    stat = {}
    for v in sorted(set(my_views)):
        st = r.render_into(cams[v], outs, stats=True)
        stat[v] = (int(st.kept), int(st.bin_entries), int(st.tiles), int(st.exact_items),
                   int(st.resolves))
    need = max(s_[1] for s_ in stat.values())
    r.ws.ensure(gs.n, W, H, int(need * 1.1) + 4096)

    # views in flight: one (stream, workspace, output buffers) per slot
    from paper_2402_00525_b200.renderer import Workspace
    n_str = max(1, args.streams)
    streams = [torch.cuda.current_stream(dev)] + [torch.cuda.Stream(dev) for _ in range(n_str - 1)]
    wss, c_outs, keep = [r.ws], [r.outputs_struct(outs)], [outs]
    for _ in range(n_str - 1):
        w_ = Workspace(dev)
        w_.ensure(gs.n, W, H, int(need * 1.1) + 4096)
        o_ = r.alloc_outputs(W, H)
        wss.append(w_)
        c_outs.append(r.outputs_struct(o_))
        keep.append(o_)
    c_scene = r.c_scene
    c_cfg = make_config(cfg, mode, fast32=args.fast32)
    c_out = c_outs[0]
    c_cams = [make_camera(c) for c in cams]
    stream = streams[0]
    s_ptrs = [ctypes.c_void_p(st.cuda_stream) for st in streams]
    n_ev = 5 * steps + 2
    ev = (ctypes.c_void_p * n_ev)()
    assert lib.stp_events_create(n_ev, ev) == 0

    def one(v, events=None, slot=0):
        ws_ = wss[slot]
        if events is None:
            rc = lib.stp_render(ctypes.byref(c_scene), ctypes.byref(c_cams[v]), ctypes.byref(c_cfg),
                                ctypes.c_void_p(ws_.ptr), ws_.nbytes, ctypes.byref(c_outs[slot]),
                                None, s_ptrs[slot])
        else:
            rc = lib.stp_render_events(ctypes.byref(c_scene), ctypes.byref(c_cams[v]),
                                       ctypes.byref(c_cfg), ctypes.c_void_p(ws_.ptr), ws_.nbytes,
                                       ctypes.byref(c_outs[slot]), events, s_ptrs[slot])
        if rc != 0:
            raise RuntimeError(f"stp_render failed: {_lib.error_string(rc)}")

    for s in range(warm):
        one(my_views[s], slot=s % n_str)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    time.sleep(0.25)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    # stage events of every timed view on its own stream; the region runs from
    # an event on stream 0 that every stream waits for to an event on stream 0
    # that waits for every stream
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(streams[0])
    for st in streams[1:]:
        st.wait_event(t_start)
    for s in range(steps):
        evs = (ctypes.c_void_p * 5)(*ev[5 * s: 5 * s + 5])
        one(my_views[warm + s], evs, slot=s % n_str)
    for st in streams[1:]:
        j = torch.cuda.Event()
        j.record(st)
        streams[0].wait_event(j)
    t_end.record(streams[0])
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    clk = clocks.stop()

    def el(a, b):
        ms = ctypes.c_float()
        assert lib.stp_event_elapsed_ms(ctypes.c_void_p(a), ctypes.c_void_p(b), ctypes.byref(ms)) == 0
        return ms.value

    total_ms = t_start.elapsed_time(t_end)
    if n_str > 1:
        # with several views in flight the per-view stage events overlap: the
        # per-kernel times (stage_ms, roofline) come from a separate pass with
        # one view at a time on stream 0 (outside the timed region)
        n_stage = min(steps, 16)
        for s in range(n_stage):
            evs = (ctypes.c_void_p * 5)(*ev[5 * s: 5 * s + 5])
            one(my_views[warm + s], evs, slot=0)
        torch.cuda.synchronize()
    else:
        n_stage = steps
    stage = np.array([[el(ev[5 * s + i], ev[5 * s + i + 1]) for i in range(4)]
                      for s in range(n_stage)])
    lib.stp_events_destroy(n_ev, ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * steps / (max_ms / 1e3)

    # roofline of the dominant kernel (K6 hierarchical render) and of the view
    stage_mean = stage.mean(axis=0)
    timed_views = my_views[warm:warm + n_stage]
    n_v = np.mean([stat[v][0] for v in timed_views])
    e = np.mean([stat[v][1] for v in timed_views])
    P = W * H
    view_b, k6_b = b_alg(gs.n, gs.sh_coeffs, n_v, e, P, cfg.with_depth)
    peak, peak_src = peaks()
    names = ["K0+K1 preprocess", "K2+K3 scan+duplicate", "K4+K5 sort+ranges", "K6 render"]
    dom = int(np.argmax(stage_mean))
    k6_ms = stage_mean[3]
    achieved = k6_b / (k6_ms / 1e3) / 1e9
    traffic = None
    gz = type(mode).__name__ == "GlobalZ"
    tr_path = os.path.join(ROOT, "profiles", "k6_traffic.json")
    if os.path.exists(tr_path) and not gz:  # the capture is of the hierarchical k_render
        try:
            with open(tr_path) as f:
                traffic = json.load(f).get("bytes_per_launch")
        except Exception:
            traffic = None

    # e2e: the public render path (Renderer.render_into, one per view slot)
    # with host output buffers (pinned): per step the camera goes host->device
    # (by-value launch params) and colour + transmittance come back
    # device->host, on the same streams / views-in-flight as the timed region.
    e2e_steps = args.e2e_steps or min(steps, 32)
    rs = [r] + [Renderer(gs, mode, cfg, dev, fast32=args.fast32) for _ in range(n_str - 1)]
    for k in range(1, n_str):
        rs[k].ws = wss[k]
    host = [(torch.empty((H, W, 3), dtype=torch.float32, pin_memory=True),
             torch.empty((H, W), dtype=torch.float32, pin_memory=True)) for _ in range(n_str)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for st in streams[1:]:
        st.wait_event(e0)
    for s in range(e2e_steps):
        k = s % n_str
        with torch.cuda.stream(streams[k]):
            rs[k].render_into(cams[my_views[warm + s % steps]], keep[k],
                              stream=streams[k].cuda_stream)
            host[k][0].copy_(keep[k]["color"], non_blocking=True)
            host[k][1].copy_(keep[k]["transmittance"], non_blocking=True)
    for st in streams[1:]:
        j = torch.cuda.Event()
        j.record(st)
        streams[0].wait_event(j)
    e1.record(streams[0])
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * e2e_steps / (float(e2e_ms.item()) / 1e3)

    # K0, K1 + row count, 3 x K2, K3 + row duplicate, K4 histogram + passes,
    # K5 (ranges with the tie fix-up), K6 (fast + list pass)
    launches_per_view = (1 + 2 + 3 + 2 + 1 + r.ws.layout(gs.n, W, H).sort_passes + 1 +
                         (2 if args.fast32 and not gz else 1))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": max_ms / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 geometry/decisions + f32 blend",
        "data": "synthetic (seeded scene generator, paper_2402_00525_b200/scenes.py)",
        "config": {"workload": WORKLOADS[args.config.upper()], "gaussians": gs.n, "sh_degree": int(round(gs.sh_coeffs ** 0.5)) - 1, "width": W,
                   "height": H, "views": n_views, "views_per_step_per_gpu": 1,
                   "parallelism": f"views sharded over {world} GPU(s), no hot-path collective; "
                                  f"{n_str} views in flight per GPU (streams)",
                   "mode": mode_name(mode), "l2": "inputs larger than L2 "
                   f"(scene {sum(x.numel() for x in dev_t.values()) * 4 / 1e6:.0f} MB > 126 MB)",
                   "mean_kept": float(n_v), "mean_entries": float(e),
                   "k6_path": "fp32-state certified + float64 list pass" if args.fast32
                   else "float64",
                   "mean_exact_items": float(np.mean([stat[v][3] for v in timed_views])),
                   "mean_resolves": float(np.mean([stat[v][4] for v in timed_views]))},
        "stage_ms": {nm: float(x) for nm, x in zip(names, stage_mean)},
        "stage_ms_note": "one view at a time (CUDA events per stage)" + (
            f"; the timed region runs {n_str} views in flight" if n_str > 1 else ""),
        "roofline": {"bound": "hbm",
                     "kernel": "K6 render (k_render_globalz)" if gz else "K6 render (k_render)",
                     "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": float(k6_b),
                     "dominant_stage": names[dom]},
        "view_roofline": {"achieved": view_b / (max_ms / steps / 1e3) / 1e9, "peak": peak,
                          "unit": "GB/s", "frac": view_b / (max_ms / steps / 1e3) / 1e9 / peak,
                          "algorithmic_bytes_per_view": float(view_b)},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": ctypes.sizeof(_lib.StpCamera),
                "d2h_bytes_per_step": H * W * 16, "steps": e2e_steps},
        "gpu_launches": launches_per_view * steps,
        "clocks": clk,
        "wall_s_timed_region": t_wall,
        "scene_setup_s": t_gen,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        host = {k: dev_t[k].cpu().numpy() for k in keys}
        rate, done, times = cpu_view_rate(host, cams, [my_views[warm]] * 3, 30.0, threads)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{done} full {args.config.upper()} view(s) (view {my_views[warm]}): "
                                          "project + bin_and_sort + hierarchical render of "
                                          "all tiles by the float64 C++ restatement "
                                          "(oracle/stp_oracle.cpp)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
