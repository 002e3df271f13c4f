"""Multi-GPU view sharding: one process per GPU, camera views partitioned
across ranks, no collective on the hot path.

The reference renders a trajectory as a sequential loop of independent
``render`` calls (rasterizer.py:758-772); views share nothing but the scene,
so they shard with no exchange.  Each rank holds a replica of the scene
(broadcast once from rank 0 by ``replicate_scene``), renders the contiguous
block of views ``shard_views`` assigns it, and -- only when asked -- the
framebuffers are gathered to rank 0 (``gather_frames``; NCCL over NVLink on
the GPU box, gloo in the CPU tests).

``render_fn(cam, view_index) -> dict of tensors`` is the per-view renderer;
the default is the device Renderer (C ABI -> sm_100a kernels).  Tests inject
a CPU checker to exercise the distributed plumbing without a GPU.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist

SCENE_KEYS = ("means", "quats", "scales", "opacity", "sh")


def shard_views(n_views: int, world: int, rank: int) -> list[int]:
    """View v goes to rank v * world // n_views (contiguous blocks, sizes
    differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    lo = (rank * n_views + world - 1) // world
    hi = ((rank + 1) * n_views + world - 1) // world
    return list(range(lo, hi))


def owner_of(view: int, n_views: int, world: int) -> int:
    return view * world // n_views


def replicate_scene(scene: dict | None, device, src: int = 0, group=None) -> dict:
    """Broadcast the scene tensors from ``src`` to every rank (once per
    scene, not per view).  ``scene`` is only read on ``src``."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return {k: torch.as_tensor(scene[k], dtype=torch.float32).to(device).contiguous()
                for k in SCENE_KEYS}
    meta = [None]
    if rank == src:
        meta = [[tuple(torch.as_tensor(scene[k]).shape) for k in SCENE_KEYS]]
    dist.broadcast_object_list(meta, src=src, group=group)
    out = {}
    for k, shp in zip(SCENE_KEYS, meta[0]):
        if rank == src:
            t = torch.as_tensor(scene[k], dtype=torch.float32).to(device).contiguous()
        else:
            t = torch.empty(shp, dtype=torch.float32, device=device)
        dist.broadcast(t, src=src, group=group)
        out[k] = t
    return out


def render_shard(cams: Sequence, render_fn: Callable, world: int | None = None,
                 rank: int | None = None) -> dict[int, dict]:
    """Render this rank's views; returns {view_index: frame dict}."""
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    return {v: render_fn(cams[v], v) for v in shard_views(len(cams), world, rank)}


def gather_frames(local: dict[int, dict], n_views: int, keys=("color", "transmittance"),
                  dst: int = 0, group=None):
    """Optional framebuffer gather to ``dst`` (the only collective, off the
    hot path).  Every rank sends its views in order with point-to-point
    transfers; returns {view: {key: tensor}} on ``dst`` and None elsewhere."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return {v: {k: f[k] for k in keys} for v, f in local.items()}
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if rank != dst:
        for v in sorted(local):
            for k in keys:
                dist.send(local[v][k].contiguous(), dst=dst, group=group)
        return None
    out = {v: {k: local[v][k] for k in keys} for v in local}
    any_frame = next(iter(local.values()), None)
    for r in range(world):
        if r == dst:
            continue
        for v in shard_views(n_views, world, r):
            out[v] = {}
            for k in keys:
                proto = any_frame[k] if any_frame is not None else None
                if proto is None:
                    raise RuntimeError("gather_frames: destination rank rendered no view")
                buf = torch.empty_like(proto)
                dist.recv(buf, src=r, group=group)
                out[v][k] = buf
    return out


def render_shard_streamed(cams: Sequence, render_fn: Callable, finalize_fn: Callable | None = None,
                          keys=("color", "transmittance"), dst: int = 0, gather: bool = True,
                          group=None) -> dict[int, dict] | None:
    """Render this rank's views and stream every finished frame to ``dst``
    while the next view renders (the optional gather,
    overlapped).  ``render_fn(cam, v)`` enqueues view v and returns its frame
    dict without synchronising; ``finalize_fn(v, frame)`` is called one view
    later (after the next view is enqueued) and returns the checked frame --
    the device renderer reads the view's status word there and re-renders an
    overflowed view.  Frames are sent with point-to-point isend / irecv
    (NCCL on the GPU box: the transfer runs on NCCL's stream behind the
    render work already enqueued).  Returns {view: frame} on ``dst`` (every
    view when ``gather``) and this rank's frames elsewhere."""
    finalize_fn = finalize_fn or (lambda v, f: f)
    n = len(cams)
    on = dist.is_initialized() and dist.get_world_size(group) > 1
    world = dist.get_world_size(group) if on else 1
    rank = dist.get_rank(group) if on else 0
    mine = shard_views(n, world, rank)
    out: dict[int, dict] = {}
    works = []
    pending = None

    def ship(v, frame):
        out[v] = frame
        if on and gather and rank != dst:
            for k in keys:
                works.append(dist.isend(frame[k].contiguous(), dst=dst, group=group))

    for v in mine:
        frame = render_fn(cams[v], v)
        if pending is not None:
            ship(pending[0], finalize_fn(*pending))
        pending = (v, frame)
    if pending is not None:
        ship(pending[0], finalize_fn(*pending))
    if on and gather and rank == dst:
        proto = next(iter(out.values()), None)
        for r in range(world):
            if r == dst:
                continue
            for v in shard_views(n, world, r):
                if proto is None:
                    raise RuntimeError("render_shard_streamed: destination rank rendered no view")
                out[v] = {k: torch.empty_like(proto[k]) for k in keys}
                for k in keys:
                    works.append(dist.irecv(out[v][k], src=r, group=group))
    for w in works:
        w.wait()
    return out


def device_render_fn(scene: dict, mode=None, cfg=None, device=None) -> Callable:
    """Per-view renderer on this rank's GPU (no CPU fallback): returns
    float32 device tensors (synchronous: stats + overflow retry)."""
    from .renderer import GaussianScene, Renderer
    gs = GaussianScene(*(scene[k] for k in SCENE_KEYS), device=device)
    r = Renderer(gs, mode, cfg, gs.device)

    def fn(cam, v):
        outs = r.alloc_outputs(cam.width, cam.height)
        r.render_into(cam, outs, stats=True)
        return outs

    return fn


def device_streamed_fns(scene: dict, mode=None, cfg=None, device=None):
    """(render_fn, finalize_fn) for ``render_shard_streamed`` on this rank's
    GPU: asynchronous views (stp_render, stats = NULL) with a status word
    per view, checked one view later; an overflowed view is re-rendered
    synchronously after the workspace grows."""
    from .renderer import GaussianScene, Renderer
    gs = scene if isinstance(scene, GaussianScene) else \
        GaussianScene(*(scene[k] for k in SCENE_KEYS), device=device)
    r = Renderer(gs, mode, cfg, gs.device)

    def render_fn(cam, v):
        outs = r.alloc_outputs(cam.width, cam.height)
        outs["status"] = torch.zeros(2, dtype=torch.int64, device=gs.device)
        r.render_into(cam, outs)
        return outs

    def finalize_fn(v, outs):
        st = outs.pop("status")
        if not r.check_status(st):
            r.render_into(cam_of[v], outs, stats=True)
        return outs

    cam_of: dict = {}

    def render_fn_keep(cam, v):
        cam_of[v] = cam
        return render_fn(cam, v)

    return render_fn_keep, finalize_fn


# ---------------------------------------------------------------------------
# One view split across GPUs (the C4 latency option): every
# rank runs K1-K5 for the whole view (redundant, cheap next to K6) and K6 for
# a band of tile rows; the bands are then all-gathered so every rank (or rank
# 0) holds the frame.  The band is the only exchange and happens after the
# render, not inside it.

def band_rows(grid_h: int, world: int, rank: int) -> tuple[int, int]:
    """Tile rows [r0, r1) of ``rank``: contiguous, sizes differ by at most one."""
    return (rank * grid_h) // world, ((rank + 1) * grid_h) // world


def band_tiles(grid_w: int, grid_h: int, world: int, rank: int) -> tuple[int, int]:
    """Row-major tile ids [t0, t1) of ``rank``'s band (whole tile rows)."""
    r0, r1 = band_rows(grid_h, world, rank)
    return r0 * grid_w, r1 * grid_w


def gather_band_frame(outs: dict, width: int, height: int, world: int, rank: int,
                      tile: int = 16, group=None, keys=("color", "transmittance", "depth")) -> dict:
    """All-gather the band pixels rendered by each rank into full frames
    (in place in ``outs``).  Bands are whole tile rows, i.e. contiguous
    image rows [16 r0, min(16 r1, H))."""
    gh = (height + tile - 1) // tile
    if not dist.is_initialized() or world == 1:
        return outs
    for k in keys:
        t = outs.get(k)
        if t is None:
            continue
        rows = [(min(band_rows(gh, world, q)[0] * tile, height),
                 min(band_rows(gh, world, q)[1] * tile, height)) for q in range(world)]
        # all_gather needs equal sizes: pad every band to the largest
        hmax = max(b - a for a, b in rows)
        shape = (hmax,) + tuple(t.shape[1:])
        a, b = rows[rank]
        mine = torch.zeros(shape, dtype=t.dtype, device=t.device)
        mine[: b - a] = t[a:b]
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        for q, (a, b) in enumerate(rows):
            t[a:b] = parts[q][: b - a]
    return outs
