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

``--gpus N`` without a torchrun environment spawns N ranks itself (one
process per GPU, 127.0.0.1 rendezvous); under torchrun WORLD_SIZE must equal
N.  Prints ONE JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
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
    "C5": "C5: synthetic 1.5M half-density scene (SH3), 1080p fixed-position yaw sweep",
}
KERNELS = ("K0 init", "K1 preprocess", "K2 scan", "K3 duplicate", "K4 sort", "K5 ranges",
           "K6 render")
STAGES = ("K0+K1 preprocess", "K2+K3 scan+duplicate", "K4+K5 sort+ranges", "K6 render")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=128)
    p.add_argument("--warmup", type=int, default=8)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="C3")
    p.add_argument("--mode", default="hierarchical",
                   help="sort mode: hierarchical (the paper's pipeline, default), globalz "
                        "(the 3DGS baseline order), full, window:k")
    p.add_argument("--gaussians", type=int, default=None, help="override N (debug)")
    p.add_argument("--views", type=int, default=256)
    p.add_argument("--no-cpu-baseline", action="store_true")
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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


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


def kernel_bytes(n, sh_k, n_v, e, p, n_tiles, with_depth=False):
    """Algorithmic HBM bytes per launch of each kernel (80 B
    splat record written once / read once, a 12 B (key, value) entry pair
    touched 4x, 16-20 B per output pixel)."""
    out_px = 20 if with_depth else 16
    return {
        "K0 init": 8 * n_tiles,                                   # tile ranges reset
        "K1 preprocess": n * 4 * (11 + 3 * sh_k) + 80 * n_v + 4 * n,   # scene read, record + count write
        "K2 scan": 8 * n,                                         # counts read, offsets write
        "K3 duplicate": 80 * n_v + 12 * e,                        # record read, entry write
        "K4 sort": 24 * e,                                        # entries read + written once
        "K5 ranges": 12 * e + 8 * n_tiles,                        # sorted keys read, ids + ranges written
        "K6 render": 80 * n_v + 12 * e + out_px * p,              # records + entries read, pixels written
    }


def view_bytes(n, sh_k, n_v, e, p, with_depth=False):
    """SURVEY.md 8(d) B_alg of one view."""
    out_px = 20 if with_depth else 16
    return n * 4 * (11 + 3 * sh_k) + 2 * 80 * n_v + 48 * e + out_px * p


def config_dict(args, n, W, H, n_views, mode_nm):
    """The same config for both arms (the driver compares them)."""
    return {"workload": WORKLOADS[args.config.upper()], "gaussians": int(n), "width": int(W),
            "height": int(H), "views": int(n_views), "mode": mode_nm,
            "views_per_step_per_gpu": 1,
            "l2": "inputs larger than L2 (scene > 126 MB, per-view records/entries > 126 MB)"}


# ----------------------------------------------------------------------------
# reference arm: the reference's algorithm on the host cores (oracle port)

def cpu_view_rate(scene, cams, views, budget_s, threads, mode=None, keep_first=False):
    """Full views (project + bin_and_sort + render of every tile under the
    sort mode, hierarchical by default) of the C++ restatement of the
    reference, all host threads."""
    import oracle
    from paper_2402_00525_b200 import Hierarchical, RenderConfig
    mode = mode if mode is not None else Hierarchical()
    times, first = [], None
    t_all = time.perf_counter()
    for v in views:
        t0 = time.perf_counter()
        out = oracle.render(scene, cams[v], RenderConfig(), mode, threads=threads)
        times.append(time.perf_counter() - t0)
        if keep_first and first is None:
            first = out
        if time.perf_counter() - t_all > budget_s:
            break
    return len(times) / sum(times), len(times), times, first


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2402_00525_b200 import scenes
    from paper_2402_00525_b200.types import mode_name, parse_mode
    scene, cams = scenes.config_scene(args.config, n=args.gaussians, n_views=args.views)
    threads = host_threads()
    mode = parse_mode(args.mode)
    warm = min(args.warmup, 2)
    if warm:
        cpu_view_rate(scene, cams, list(range(warm)), 1e9, threads, mode)   # bounded warmup
    # the views our arm times: rank 0's views after its warmup
    views = [(args.warmup + s) * args.gpus % len(cams) for s in range(args.steps)]
    rate, done, times, _ = cpu_view_rate(scene, cams, views, args.cpu_seconds, threads, mode)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": ws,
        "steps": done, "warmup": warm, "ms_per_step": 1e3 / rate,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded scene generator, paper_2402_00525_b200/scenes.py)",
        "config": config_dict(args, len(scene["opacity"]), cams[0].width, cams[0].height,
                              len(cams), mode_name(mode)),
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

def _profile_json(name):
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def frame_parity(r, gpu_out, cam, ref):
    """GPU frame (benched path) vs the oracle frame of the same view."""
    tile, gid, _ = r.debug_bins(cam)
    src = ref["batch"].source_index
    rank = np.searchsorted(src, gid)
    t_ref, s_ref = ref["bins"][0], ref["bins"][1]
    tiles_equal = bool(len(tile) == len(t_ref) and np.array_equal(tile, t_ref))
    order_equal = bool(tiles_equal and np.array_equal(rank, s_ref))
    col = gpu_out["color"].double().cpu().numpy()
    tn = gpu_out["transmittance"].double().cpu().numpy()
    return {"max_abs_color": float(np.abs(col - ref["color"]).max()),
            "max_abs_transmittance": float(np.abs(tn - ref["transmittance"]).max()),
            "tiles_equal": tiles_equal, "order_equal": order_equal,
            "entries": int(len(t_ref)), "pixels": int(col.shape[0] * col.shape[1]),
            "tolerance": 1e-4,
            "pass": bool(tiles_equal and order_equal and
                         float(np.abs(col - ref["color"]).max()) <= 1e-4 and
                         float(np.abs(tn - ref["transmittance"]).max()) <= 1e-4)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2402_00525_b200 import RenderConfig, _lib, scenes
    from paper_2402_00525_b200.renderer import (GaussianScene, Renderer, Workspace, make_camera,
                                                make_config)
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
    r = Renderer(gs, mode, cfg, dev)
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
        stat[v] = (int(st.kept), int(st.bin_entries), int(st.tiles), int(st.tie_runs))
    need = max(s_[1] for s_ in stat.values())
    r.ws.ensure(gs.n, W, H, int(need * 1.1) + 4096)

    # views in flight: one (stream, workspace, output buffers, status word) per slot
    n_str = max(1, args.streams)
    streams = [torch.cuda.current_stream(dev)] + [torch.cuda.Stream(dev) for _ in range(n_str - 1)]
    wss, c_outs, keep = [r.ws], [], [outs]
    for _ in range(n_str - 1):
        w_ = Workspace(dev)
        w_.ensure(gs.n, W, H, int(need * 1.1) + 4096)
        wss.append(w_)
        keep.append(r.alloc_outputs(W, H))
    # per-step device status words (StpOutputs.status): every timed frame's
    # overflow report, checked after the timed region
    status = torch.zeros((steps + warm, 2), dtype=torch.int64, device=dev)
    for k in range(n_str):
        c_outs.append(r.outputs_struct(keep[k]))
    c_scene = r.c_scene
    c_cfg = make_config(cfg, mode)
    c_cams = [make_camera(c) for c in cams]
    s_ptrs = [ctypes.c_void_p(st.cuda_stream) for st in streams]
    NE = _lib.STP_KERNEL_EVENTS
    n_ev = NE * min(steps, 16)
    ev = (ctypes.c_void_p * n_ev)()
    assert lib.stp_events_create(n_ev, ev) == 0
    launches = [0]

    def one(v, step, slot=0, events=None):
        co = c_outs[slot]
        co.status = status[step].data_ptr()
        ws_ = wss[slot]
        if events is None:
            rc = lib.stp_render(ctypes.byref(c_scene), ctypes.byref(c_cams[v]), ctypes.byref(c_cfg),
                                ctypes.c_void_p(ws_.ptr), ws_.nbytes, ctypes.byref(co),
                                None, s_ptrs[slot])
        else:
            rc = lib.stp_render_events(ctypes.byref(c_scene), ctypes.byref(c_cams[v]),
                                       ctypes.byref(c_cfg), ctypes.c_void_p(ws_.ptr), ws_.nbytes,
                                       ctypes.byref(co), events, NE, s_ptrs[slot])
        if rc != 0:
            raise RuntimeError(f"stp_render failed: {_lib.error_string(rc)}")

    for s in range(warm):
        one(my_views[s], s, slot=s % n_str)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    time.sleep(0.25)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    # the region runs from an event on stream 0 that every stream waits for
    # to an event on stream 0 that waits for every stream
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(streams[0])
    for st in streams[1:]:
        st.wait_event(t_start)
    for s in range(steps):
        one(my_views[warm + s], warm + s, slot=s % n_str)
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
    st_codes = status[:, 0].cpu().numpy()
    if (st_codes != 0).any():
        raise RuntimeError(f"timed frames reported status {sorted(set(st_codes.tolist()))} "
                           "(entry overflow): the measurement is invalid")

    def el(a, b):
        ms = ctypes.c_float()
        assert lib.stp_event_elapsed_ms(ctypes.c_void_p(a), ctypes.c_void_p(b), ctypes.byref(ms)) == 0
        return ms.value

    total_ms = t_start.elapsed_time(t_end)
    # per-kernel times (CUDA events at every kernel boundary, on the launching
    # stream): a separate pass with one view at a time outside the timed
    # region, because with several views in flight the intervals overlap
    n_stage = min(steps, 16)
    for s in range(n_stage):
        evs = (ctypes.c_void_p * NE)(*ev[NE * s: NE * s + NE])
        one(my_views[warm + s], warm + s, slot=0, events=evs)
    torch.cuda.synchronize()
    kms = np.array([[el(ev[NE * s + i], ev[NE * s + i + 1]) for i in range(NE - 1)]
                    for s in range(n_stage)])
    lib.stp_events_destroy(n_ev, ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * steps / (max_ms / 1e3)

    # rooflines: per kernel (algorithmic bytes / event-timed duration) and the view
    kmean = kms.mean(axis=0)
    stage_mean = [kmean[0] + kmean[1], kmean[2] + kmean[3], kmean[4] + kmean[5], kmean[6]]
    timed_views = my_views[warm:warm + n_stage]
    n_v = float(np.mean([stat[v][0] for v in timed_views]))
    e = float(np.mean([stat[v][1] for v in timed_views]))
    P = W * H
    L = r.ws.layout(gs.n, W, H)
    kb = kernel_bytes(gs.n, gs.sh_coeffs, n_v, e, P, L.n_tiles, cfg.with_depth)
    vb = view_bytes(gs.n, gs.sh_coeffs, n_v, e, P, cfg.with_depth)
    peak, peak_src = peaks()
    ncu = _profile_json("ncu_kernels.json") or {}
    gz = type(mode).__name__ == "GlobalZ"
    per_kernel = {}
    for name, ms in zip(KERNELS, kmean):
        a = kb[name] / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        d = {"ms": float(ms), "algorithmic_bytes": float(kb[name]), "achieved": a,
             "frac": a / peak, "share_of_view": float(ms / kmean.sum())}
        cap = ncu.get("kernels", {}).get(name)
        if cap and (not gz or name != "K6 render"):
            d["traffic"] = cap.get("dram_bytes_per_view")
            for k2 in ("issue_active_frac", "fp64_pipe_frac", "achieved_occupancy", "top_stalls",
                       "dram_frac_of_peak_ncu"):
                if k2 in cap:
                    d[k2] = cap[k2]
        per_kernel[name] = d
    k6 = per_kernel["K6 render"]
    dom = max(per_kernel, key=lambda k_: per_kernel[k_]["ms"])

    # e2e: the public render path (Renderer.render_into, one per view slot)
    # with host output buffers (pinned): per step the camera goes host->device
    # (by-value launch params) and colour + transmittance + the status word
    # come back device->host.  The device->host copies run on their own
    # stream (the copy engine) behind an event of the view that produced
    # them, so they overlap the next views' kernels; every view slot has two
    # output buffers, and a slot waits for the copy of the buffer it is about
    # to overwrite (two views earlier).  Every step's status is checked.
    e2e_steps = args.e2e_steps or min(steps, 32)
    rs = [r] + [Renderer(gs, mode, cfg, dev) for _ in range(n_str - 1)]
    for k in range(1, n_str):
        rs[k].ws = wss[k]
    bufs = [[keep[k], r.alloc_outputs(W, H)] for k in range(n_str)]
    for k in range(n_str):
        for b in bufs[k]:
            b["status"] = torch.zeros(2, dtype=torch.int64, device=dev)
    host = [[(torch.empty((H, W, 3), dtype=torch.float32, pin_memory=True),
              torch.empty((H, W), dtype=torch.float32, pin_memory=True)) for _ in range(2)]
            for _ in range(n_str)]
    host_status = torch.zeros((e2e_steps, 2), dtype=torch.int64, pin_memory=True)
    copy_stream = torch.cuda.Stream(dev)
    copied = [[None, None] for _ in range(n_str)]

    def e2e_step(s, view):
        k = s % n_str
        pb = (s // n_str) & 1
        o = bufs[k][pb]
        if copied[k][pb] is not None:
            streams[k].wait_event(copied[k][pb])
        with torch.cuda.stream(streams[k]):
            rs[k].render_into(cams[view], o, stream=streams[k].cuda_stream)
        done = torch.cuda.Event()
        done.record(streams[k])
        copy_stream.wait_event(done)
        with torch.cuda.stream(copy_stream):
            host[k][pb][0].copy_(o["color"], non_blocking=True)
            host[k][pb][1].copy_(o["transmittance"], non_blocking=True)
            host_status[s % e2e_steps].copy_(o["status"], non_blocking=True)
        c = torch.cuda.Event()
        c.record(copy_stream)
        copied[k][pb] = c

    # untimed warm-up of every (view slot, buffer) pair: renderers, output
    # buffers, pinned host buffers and the copy stream see their first use here
    for s in range(2 * n_str):
        e2e_step(s, my_views[s % len(my_views)])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for st in streams[1:] + [copy_stream]:
        st.wait_event(e0)
    for s in range(e2e_steps):
        e2e_step(s, my_views[warm + s % steps])
    for st in streams[1:]:
        j = torch.cuda.Event()
        j.record(st)
        copy_stream.wait_event(j)
    streams[0].wait_stream(copy_stream)
    e1.record(streams[0])
    torch.cuda.synchronize()
    if (host_status[:, 0] != 0).any():
        raise RuntimeError("e2e frames reported an entry overflow")
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * e2e_steps / (float(e2e_ms.item()) / 1e3)

    # launches per view: K0, K1 + K1b row count, 3 x K2, K3 + K3b, K4
    # histogram + passes, K5, K6
    launches_per_view = 1 + 2 + 3 + 2 + 1 + L.sort_passes + 1 + 1
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": max_ms / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 geometry/decisions + f32 blend",
        "data": "synthetic (seeded scene generator, paper_2402_00525_b200/scenes.py)",
        "config": config_dict(args, gs.n, W, H, n_views, mode_name(mode)),
        "workload_stats": {"sh_degree": int(round(gs.sh_coeffs ** 0.5)) - 1,
                           "mean_kept": n_v, "mean_entries": e,
                           "mean_tie_runs": float(np.mean([stat[v][3] for v in timed_views])),
                           "parallelism": f"views sharded over {world} GPU(s), no hot-path "
                                          f"collective; {n_str} views in flight per GPU (streams)"},
        "stage_ms": {nm: float(x) for nm, x in zip(STAGES, stage_mean)},
        "kernel_ms": {nm: float(x) for nm, x in zip(KERNELS, kmean)},
        "stage_ms_note": "one view at a time, CUDA events at every kernel boundary on the "
                         f"launching stream ({n_stage} views)" + (
            f"; the timed region runs {n_str} views in flight" if n_str > 1 else ""),
        "roofline": {"bound": "hbm",
                     "kernel": "K6 render (k_render_globalz)" if gz else "K6 render (k_render)",
                     "achieved": k6["achieved"], "peak": peak, "unit": "GB/s",
                     "frac": k6["achieved"] / peak, "traffic": k6.get("traffic"),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": k6["algorithmic_bytes"],
                     "dominant_kernel": dom,
                     "note": "K6 is bound by float64 dependent latency / issue, not HBM: its "
                             "issue-slot and FP64-pipe fractions (committed ncu capture) are in "
                             "per_kernel['K6 render']",
                     "per_kernel": per_kernel},
        "view_roofline": {"achieved": vb / (max_ms / steps / 1e3) / 1e9, "peak": peak,
                          "unit": "GB/s", "frac": vb / (max_ms / steps / 1e3) / 1e9 / peak,
                          "algorithmic_bytes_per_view": float(vb)},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": ctypes.sizeof(_lib.StpCamera),
                "d2h_bytes_per_step": H * W * 16 + 16, "steps": e2e_steps,
                "path": "Renderer.render_into (C ABI stp_render) -> pinned host colour + T "
                        "(copies on a copy stream, double-buffered outputs per view slot)"},
        "gpu_launches": launches_per_view * steps,
        "clocks": clk,
        "wall_s_timed_region": t_wall,
        "scene_setup_s": t_gen,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # drop-in API throughput: render(GaussianScene, cam, mode, cfg) returning
        # the reference's float64 numpy FrameOutput (allocation, sync, stats,
        # float64 conversion and D2H included)
        from paper_2402_00525_b200.renderer import render as dropin_render
        n_api = 4
        dropin_render(gs, cams[my_views[warm]], mode, cfg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(n_api):
            dropin_render(gs, cams[my_views[warm + s]], mode, cfg)
        line["e2e_render_api"] = {"value": n_api / (time.perf_counter() - t0), "unit": UNIT,
                                  "steps": n_api, "timer": "host wall clock",
                                  "path": "paper_2402_00525_b200.render (drop-in), float64 "
                                          "numpy outputs"}
        # CPU baseline on the host cores, and parity of the benched frame:
        # the same view rendered by the benched path and by the oracle
        threads = host_threads()
        host_sc = {k: dev_t[k].cpu().numpy() for k in keys}
        v0 = my_views[warm]
        rate, done, times, ref = cpu_view_rate(host_sc, cams, [v0] * 3, 30.0, threads, mode,
                                               keep_first=True)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{done} full {args.config.upper()} view(s) (view {v0}): "
                                          f"project + bin_and_sort + {mode_name(mode)} render "
                                          "of all tiles by the float64 C++ restatement "
                                          "(oracle/stp_oracle.cpp)"}
        # the unmodified reference (baseline/_ref) itself, measured on this
        # box's host by scripts/reference_cpu_point.py (SURVEY.md 8(d)
        # protocol: projection and bin_and_sort in full, render_tile on a
        # stratified tile sample, extrapolated by entries) -- too slow to
        # re-run inside every bench (minutes per view)
        refpt = _profile_json(f"reference_python_{args.config.upper()}.json")
        if refpt and type(mode).__name__ == "Hierarchical":
            line["cpu_baseline"]["reference_python"] = {
                "value": refpt["views_per_s"], "unit": UNIT, "cores": refpt["workers"],
                "kind": "reference", "s_per_view": refpt["s_per_view"],
                "sample": f"view {refpt['view']}: project_scene + bin_and_sort in full, "
                          f"hierarchy.render_tile on {refpt['tiles_sampled']} stratified tiles "
                          f"({refpt['entries_sampled']} of {refpt['bin_entries']} entries), "
                          "extrapolated by entries; 1 worker (GIL-bound pool)",
                "source": f"profiles/reference_python_{args.config.upper()}.json"}
        pouts = r.alloc_outputs(W, H)
        r.render_into(cams[v0], pouts)
        torch.cuda.synchronize()
        if not r.check_status():
            raise RuntimeError("parity frame overflowed")
        line["parity"] = dict(frame_parity(r, pouts, cams[v0], ref), view=int(v0),
                              path="stp_render (benched kernels) vs oracle/stp_oracle.cpp")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawned(local_rank, world, port, argv):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(local_rank), LOCAL_RANK=str(local_rank),
                      LOCAL_WORLD_SIZE=str(world))
    sys.argv = argv
    main()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `--gpus N` without torchrun: one process per GPU, spawned here
        import torch.multiprocessing as mp
        mp.spawn(_spawned, args=(args.gpus, _free_port(), list(sys.argv)), nprocs=args.gpus,
                 join=True)
        return
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus and "WORLD_SIZE" in os.environ:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    run_ours(args)


if __name__ == "__main__":
    main()
