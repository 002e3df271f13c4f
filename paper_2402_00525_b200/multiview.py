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


def device_render_fn(scene: dict, mode=None, cfg=None, device=None) -> Callable:
    """Per-view renderer on this rank's GPU (no CPU fallback): returns
    float32 device tensors."""
    from .renderer import GaussianScene, Renderer
    gs = GaussianScene(*(scene[k] for k in SCENE_KEYS), device=device)
    r = Renderer(gs, mode, cfg, gs.device)

    def fn(cam, v):
        outs = r.alloc_outputs(cam.width, cam.height)
        r.render_into(cam, outs, stats=True)
        return outs

    return fn
