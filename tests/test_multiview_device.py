"""The multi-GPU view driver on the device, on the one GPU
a gpurun box has: an NCCL process group of world size 1 running the same
code the N-GPU launch runs (scene replication, view shard, streamed
framebuffer gather), plus stp_render_views (one call for a rank's views) and
the asynchronous paths' overflow status word (stp.h StpOutputs.status)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene_cams(n=60_000, views=6, w=320, h=180):
    from paper_2402_00525_b200 import scenes
    sc = scenes.to_f32_scene(scenes.garden_scene(n, 3))
    cams = scenes.orbit_cameras(views, width=w, height_px=h, f=183.0)
    return sc, cams


def _serial(sc, cams, mode=None):
    from paper_2402_00525_b200 import Hierarchical, RenderConfig
    from paper_2402_00525_b200.renderer import Renderer
    r = Renderer(sc, mode or Hierarchical(), RenderConfig())
    out = []
    for c in cams:
        o = r.alloc_outputs(c.width, c.height)
        r.render_into(c, o, stats=True)
        out.append({k: v.clone() for k, v in o.items()})
    return out


def test_nccl_world1_device_driver():
    import torch
    import torch.distributed as dist
    from paper_2402_00525_b200 import Hierarchical, RenderConfig, multiview
    sc, cams = _scene_cams()
    ref = _serial(sc, cams)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        scene_t = multiview.replicate_scene(sc, dev)
        local = multiview.render_shard(cams, multiview.device_render_fn(scene_t, Hierarchical(),
                                                                        RenderConfig(), dev))
        got = multiview.gather_frames(local, len(cams))
        rf, fin = multiview.device_streamed_fns(scene_t, Hierarchical(), RenderConfig(), dev)
        streamed = multiview.render_shard_streamed(cams, rf, fin)
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    for v in range(len(cams)):
        for k in ("color", "transmittance"):
            assert torch.equal(got[v][k], ref[v][k]), (v, k)
            assert torch.equal(streamed[v][k], ref[v][k]), (v, k)


def test_render_views_equals_serial_and_reports_overflow():
    """stp_render_views renders a rank's views in one call; with a workspace
    too small for some views their status words say WORKSPACE_TOO_SMALL and
    render_views re-renders exactly those."""
    import torch
    from paper_2402_00525_b200 import Hierarchical, RenderConfig, _lib
    from paper_2402_00525_b200.renderer import Renderer
    sc, cams = _scene_cams()
    ref = _serial(sc, cams)
    r = Renderer(sc, Hierarchical(), RenderConfig())
    outs = [r.alloc_outputs(c.width, c.height) for c in cams]
    st = r.render_views(cams, outs)
    assert (st[:, 0] == 0).all()
    for v in range(len(cams)):
        assert torch.equal(outs[v]["color"], ref[v]["color"])
    # too small: capacity below the smallest view's entries
    ents = [int(x) for x in st[:, 1].tolist()]
    r2 = Renderer(sc, Hierarchical(), RenderConfig(), entry_capacity=min(ents) // 2)
    outs2 = [r2.alloc_outputs(c.width, c.height) for c in cams]
    st2 = r2.render_views(cams, outs2, retry=False)
    torch.cuda.synchronize()
    codes = st2[:, 0].tolist()
    assert all(c == _lib.STP_ERR_WORKSPACE_TOO_SMALL for c in codes)
    assert st2[:, 1].tolist() == ents
    r3 = Renderer(sc, Hierarchical(), RenderConfig(), entry_capacity=sorted(ents)[2] + 10)
    outs3 = [r3.alloc_outputs(c.width, c.height) for c in cams]
    st3 = r3.render_views(cams, outs3)          # retries the overflowed views
    assert (st3[:, 0] == 0).all()
    for v in range(len(cams)):
        assert torch.equal(outs3[v]["color"], ref[v]["color"]), v


def test_async_overflow_status_and_retry():
    """stp_render with stats = NULL and a too-small workspace: the frame's
    status word reports the overflow and its entry count; check_status grows
    the workspace and the re-render equals the synchronous frame."""
    import torch
    from paper_2402_00525_b200 import Hierarchical, RenderConfig, _lib
    from paper_2402_00525_b200.renderer import Renderer
    sc, cams = _scene_cams(views=2)
    ref = _serial(sc, cams[:1])[0]
    r = Renderer(sc, Hierarchical(), RenderConfig(), entry_capacity=1000)
    o = r.alloc_outputs(cams[0].width, cams[0].height)
    r.render_into(cams[0], o)
    torch.cuda.synchronize()
    code, ents = r.status.tolist()
    assert code == _lib.STP_ERR_WORKSPACE_TOO_SMALL and ents > 1000
    assert not r.check_status()          # grows the workspace
    r.render_into(cams[0], o)
    assert r.check_status()
    assert torch.equal(o["color"], ref["color"])
    assert torch.equal(o["transmittance"], ref["transmittance"])
