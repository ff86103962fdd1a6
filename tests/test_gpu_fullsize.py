"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* configs[1] (the bench workload: ~10M-triangle gyroid, 1024x1024, 16 spp in one batch,
  shadows + AO) at N=1: EVERY event code and occlusion bit of the frame bit-exact against
  the oracle's full-frame render, pixels within the north_star tolerance, ray counts equal.
* configs[1] split over 4 ranks (loopback group, spp batches of 4): routing matrices S,
  visits V and step counts bit-exact against the oracle's routing simulator, full frame.
* configs[2] (1024^3 float32 volume in bricks, 1920x1080, DVR + volume shadows): sampled
  pixels (the oracle evaluates any pixel subset exactly: paths are Philox-keyed).
* the NCCL code path (DPR_FORCE_NCCL=1 makes a single rank use NCCL collectives).
"""
import os

import numpy as np
import pytest

import dpr_inputs as di
from tests.gpu_helpers import assert_parity, assert_pixels_close, gpu_render, oracle_render

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2_scene():
    return di.config2(nranks=1)


def test_config2_full_frame_single_rank(c2_scene):
    sc = c2_scene
    g = gpu_render(sc.parts, 1, sc.camera, sc.frame)
    o = oracle_render(sc.parts, 1, sc.camera, sc.frame, dp=False)
    assert_parity(g, o, check_routing=False)
    assert g[3]["steps"] == 2


def test_config2_full_frame_four_ranks():
    sc = di.config2(nranks=4, spp_batch=4)
    g = gpu_render(sc.parts, 4, sc.camera, sc.frame)
    o = oracle_render(sc.parts, 4, sc.camera, sc.frame, dp=True)
    assert_parity(g, o)
    assert o.S.sum() > 1_000_000


def test_config3_full_size_sampled():
    sc = di.config3(nranks=1)
    # GPU: whole frame; oracle: 400 random pixels (+ the centre row segment)
    g = gpu_render(sc.parts, 1, sc.camera, sc.frame)
    P = sc.frame.W * sc.frame.H
    rng = np.random.default_rng(3)
    pix = np.unique(np.concatenate([rng.choice(P, 400, replace=False),
                                    (sc.frame.H // 2) * sc.frame.W + np.arange(800, 1120)]))
    o = oracle_render(sc.parts, 1, sc.camera, sc.frame, pixels=pix, dp=False)
    ev = g[1][:, :, pix]
    oc = g[2][:, :, pix]
    assert ((o.events & 0x80000000) != 0).sum() > 50
    assert np.array_equal(ev, o.events)
    assert np.array_equal(oc, o.occl)
    assert_pixels_close(g[0][pix], o.rgba)


def test_config3_delta_tracking_full_size_sampled():
    """configs[2] (1024^3 volume) with delta tracking (DPR_FLAG_DELTA): whole frame on the
    GPU, every event / occlusion bit of 2000 sampled pixels against the oracle."""
    sc = di.config3(nranks=1)
    fr = di.Frame(**{**sc.frame.__dict__, "flags": sc.frame.flags | 16})
    g = gpu_render(sc.parts, 1, sc.camera, fr)
    P = fr.W * fr.H
    pix = np.unique(np.random.default_rng(5).choice(P, 2000, replace=False))
    o = oracle_render(sc.parts, 1, sc.camera, fr, pixels=pix, dp=False)
    assert ((o.events & 0x80000000) != 0).sum() > 50
    assert np.array_equal(g[1][:, :, pix], o.events)
    assert np.array_equal(g[2][:, :, pix], o.occl)
    assert_pixels_close(g[0][pix], o.rgba)


@pytest.mark.parametrize("mode", ["sendrecv", "fused", "fused-host"])
def test_nccl_collectives_single_rank(mode, monkeypatch):
    """DPR_FORCE_NCCL=1: frame-setup allgather, counts allgather / fused step allgather,
    (empty) grouped exchange, cudaIpc export of the fused queues, the device-driven step loop
    with its mailbox step barrier (fused), and ncclReduce of framebuffer + dumps all run
    through NCCL with one rank."""
    monkeypatch.setenv("DPR_FORCE_NCCL", "1")
    monkeypatch.setenv("DPR_EXCHANGE", mode.split("-")[0])
    monkeypatch.setenv("DPR_STEP_LOOP", "host" if mode.endswith("host") else "device")
    sc = di.config1()
    parts = di.union_parts(sc.parts)
    g = gpu_render(parts, 1, sc.camera, sc.frame)
    o = oracle_render(parts, 1, sc.camera, sc.frame)
    assert_parity(g, o)


def test_fused_exchange_falls_back_to_sendrecv(monkeypatch):
    """When some rank cannot map its peers' queues (no peer access between two GPUs; injected:
    DPR_TEST_FUSED_FAIL=<rank>), every rank agrees through one allgather and the frame runs on
    the NCCL send/recv exchange instead (host step loop), with the same parity."""
    monkeypatch.setenv("DPR_FORCE_NCCL", "1")
    monkeypatch.setenv("DPR_EXCHANGE", "fused")
    monkeypatch.setenv("DPR_STEP_LOOP", "device")
    monkeypatch.setenv("DPR_TEST_FUSED_FAIL", "0")
    sc = di.config1()
    parts = di.union_parts(sc.parts)
    g = gpu_render(parts, 1, sc.camera, sc.frame, frames=2)
    o = oracle_render(parts, 1, sc.camera, sc.frame)
    assert_parity(g, o)
    assert g[3]["step_loop_device"] == 0


def test_config4_full_size_sampled():
    """configs[3] at full size on one rank (50M spheres in 1000 cluster parts + ~5M
    triangles, 1920x1080, depth 4): every event/occlusion bit of 1500 sampled pixels."""
    sc = di.config4(nranks=1)
    g = gpu_render(sc.parts, 1, sc.camera, sc.frame)
    P = sc.frame.W * sc.frame.H
    pix = np.sort(np.random.default_rng(4).choice(P, 1500, replace=False))
    o = oracle_render(sc.parts, 1, sc.camera, sc.frame, pixels=pix, dp=False)
    assert np.array_equal(g[1][:, :, pix], o.events)
    assert np.array_equal(g[2][:, :, pix], o.occl)
    assert_pixels_close(g[0][pix], o.rgba)


def test_nccl_async_error_aborts(monkeypatch):
    """dpr.h DPR_ERR_NCCL "(incl. async errors)": the NCCL waits poll ncclCommGetAsyncError;
    on an error (injected: DPR_TEST_NCCL_FAULT=1) the communicator is aborted, the render
    returns DPR_ERR_NCCL, later collectives fail the same way, and release still works."""
    from paper_2407_00179_b200 import dpr
    monkeypatch.setenv("DPR_FORCE_NCCL", "1")
    monkeypatch.setenv("DPR_TEST_NCCL_FAULT", "1")
    sc = di.config1()
    dev = dpr.Device.create(0, 1, 0)
    try:
        dev.commit_scene_parts(di.union_parts(sc.parts))
        dev.commit_world()
        dev.set_camera(sc.camera)
        dev.set_frame(sc.frame)
        for _ in range(2):
            with pytest.raises(dpr.DprError) as e:
                dev.render_frame()
            assert e.value.code == -4
    finally:
        dev.release()


def test_config5_full_size_sampled():
    """configs[4] at full size on one GPU (~100M-triangle gyroid + the 1024^3 volume in bricks,
    3840x2160, 64 spp in 16 batches of 4, depth 2): the whole frame on the GPU, every event /
    occlusion bit of 1000 sampled pixels x 64 samples against the oracle (its BVH over 100M
    triangles takes ~2 min to build on the host)."""
    from paper_2407_00179_b200 import dpr
    sc = di.config5(nranks=1)
    fr = di.Frame(**{**sc.frame.__dict__, "flags": sc.frame.flags | dpr.DPR_FLAG_DEBUG_DUMPS})
    dev = dpr.Device.create(0, 1, 0)
    try:
        for p in sc.parts:
            dev.commit_part(p)
        dev.commit_world()
        dev.set_camera(sc.camera)
        dev.set_frame(fr)
        dev.render_frame()
        rgba = dev.map_frame().reshape(-1, 4).cpu().numpy().astype(np.float64)
        P = fr.W * fr.H
        pix = np.sort(np.random.default_rng(9).choice(P, 1000, replace=False))
        import torch
        ev, oc = dev.get_debug(fr.spp, fr.max_depth, P)
        ix = torch.as_tensor(pix, device="cuda")
        # torch has no uint32 gather on CUDA: reinterpret as int32 (same bits)
        ev = ev.view(torch.int32)[:, :, ix].cpu().numpy().view(np.uint32)
        oc = oc.view(torch.int32)[:, :, ix].cpu().numpy().view(np.uint32)
        st = dev.get_stats()
    finally:
        dev.release()
    assert st["steps"] > 16
    o = oracle_render(sc.parts, 1, sc.camera, fr, pixels=pix, dp=False)
    assert ((o.events & 0x80000000) != 0).sum() > 50  # volume events present
    assert np.array_equal(ev, o.events)
    assert np.array_equal(oc, o.occl)
    assert_pixels_close(rgba[pix], o.rgba)
