"""World-size-2 CPU (gloo) tests of the multi-GPU view-sharding plumbing
(paper_2402_00525_b200/multiview.py): scene replication by broadcast, view
partition, no collective while rendering, optional framebuffer gather.

The per-view renderer is injected: here the CPU oracle (test
infrastructure), on the GPU box the device Renderer.  The check is that the
distributed result equals rendering every view serially.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_00525_b200 import multiview


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n_views,world", [(256, 1), (256, 2), (256, 8), (240, 8), (5, 8),
                                           (7, 3), (0, 2)])
def test_shard_views_partition(n_views, world):
    got = [multiview.shard_views(n_views, world, r) for r in range(world)]
    flat = [v for g in got for v in g]
    assert flat == list(range(n_views))                      # every view once, in order
    sizes = [len(g) for g in got]
    assert max(sizes) - min(sizes) <= 1
    for r, g in enumerate(got):
        assert all(multiview.owner_of(v, n_views, world) == r for v in g)


def _scene_and_cams():
    from paper_2402_00525_b200 import scenes
    sc = scenes.to_f32_scene(scenes.garden_scene(1500, 3))
    cams = scenes.orbit_cameras(6, width=64, height_px=48, f=40.0)
    return sc, cams


def _oracle_fn(scene_t):
    import oracle
    from paper_2402_00525_b200 import Hierarchical, RenderConfig
    host = {k: v.cpu().numpy() for k, v in scene_t.items()}

    def fn(cam, v):
        out = oracle.render(host, cam, RenderConfig(), Hierarchical(), threads=1)
        return {"color": torch.from_numpy(np.ascontiguousarray(out["color"], dtype=np.float32)),
                "transmittance": torch.from_numpy(
                    np.ascontiguousarray(out["transmittance"], dtype=np.float32))}
    return fn


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, cams = _scene_and_cams()
        scene_t = multiview.replicate_scene(sc if rank == 0 else None, "cpu")
        local = multiview.render_shard(cams, _oracle_fn(scene_t))
        got = multiview.gather_frames(local, len(cams))
        if rank == 0:
            q.put({v: {k: t.numpy() for k, t in f.items()} for v, f in got.items()})
        else:
            q.put(sorted(local))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_equal_serial():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered = next(r for r in res if isinstance(r, dict))
    shard1 = next(r for r in res if isinstance(r, list))
    assert shard1 == multiview.shard_views(6, 2, 1)
    sc, cams = _scene_and_cams()
    serial = _oracle_fn({k: torch.from_numpy(v) for k, v in sc.items()})
    assert sorted(gathered) == list(range(len(cams)))
    for v, cam in enumerate(cams):
        ref = serial(cam, v)
        np.testing.assert_array_equal(gathered[v]["color"], ref["color"].numpy())
        np.testing.assert_array_equal(gathered[v]["transmittance"], ref["transmittance"].numpy())
    # the scene is visible in at least some views (not a vacuous comparison)
    assert any((gathered[v]["transmittance"] < 0.999).any() for v in gathered)


@pytest.mark.parametrize("gh,world", [(68, 2), (68, 8), (135, 8), (3, 8), (1, 2)])
def test_band_partition(gh, world):
    rows = [multiview.band_rows(gh, world, r) for r in range(world)]
    assert rows[0][0] == 0 and rows[-1][1] == gh
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 1
    assert multiview.band_tiles(120, gh, world, world - 1)[1] == 120 * gh


def _band_worker(rank, world, port, q):
    """Each rank 'renders' only its band (a copy of the oracle frame inside
    the band, garbage elsewhere) and the all-gather assembles the frame."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, cams = _scene_and_cams()
        full = _oracle_fn({k: torch.from_numpy(v) for k, v in sc.items()})(cams[1], 1)
        H, W = full["transmittance"].shape
        gh = (H + 15) // 16
        r0, r1 = multiview.band_rows(gh, world, rank)
        outs = {k: torch.full_like(v, -7.0) for k, v in full.items()}
        a, b = min(16 * r0, H), min(16 * r1, H)
        for k in outs:
            outs[k][a:b] = full[k][a:b]
        multiview.gather_band_frame(outs, W, H, world, rank, keys=tuple(outs))
        q.put((rank, {k: v.numpy() for k, v in outs.items()},
               {k: v.numpy() for k, v in full.items()}))
    finally:
        dist.destroy_process_group()


def test_gloo_band_gather():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, full in res:
        for k in full:
            np.testing.assert_array_equal(got[k], full[k])


def _streamed_worker(rank, world, port, q):
    """render_shard_streamed: frames go to rank 0 by isend / irecv right
    after each view (one view of lag for the status check)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, cams = _scene_and_cams()
        scene_t = multiview.replicate_scene(sc if rank == 0 else None, "cpu")
        fin = []
        got = multiview.render_shard_streamed(cams, _oracle_fn(scene_t),
                                              finalize_fn=lambda v, f: (fin.append(v), f)[1])
        if rank == 0:
            q.put((rank, fin, {v: {k: t.numpy() for k, t in f.items()} for v, f in got.items()}))
        else:
            q.put((rank, fin, sorted(got)))
    finally:
        dist.destroy_process_group()


def test_gloo_streamed_gather_equals_serial():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_streamed_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc, cams = _scene_and_cams()
    for rank, fin, _ in res:
        assert fin == multiview.shard_views(len(cams), world, rank)   # every view finalized once
    gathered = res[0][2]
    serial = _oracle_fn({k: torch.from_numpy(v) for k, v in sc.items()})
    assert sorted(gathered) == list(range(len(cams)))
    for v, cam in enumerate(cams):
        ref = serial(cam, v)
        np.testing.assert_array_equal(gathered[v]["color"], ref["color"].numpy())
        np.testing.assert_array_equal(gathered[v]["transmittance"], ref["transmittance"].numpy())
