"""Boundary behaviour on the GPU (include/dpr.h error contract and P:379-431 semantics)."""
import numpy as np
import pytest

import dpr_inputs as di

pytestmark = pytest.mark.gpu


def _dpr():
    from paper_2407_00179_b200 import dpr
    return dpr


def test_state_errors_and_invalid_index():
    dpr = _dpr()
    dev = dpr.Device.create(0, 1, 0)
    try:
        with pytest.raises(dpr.DprError) as e:
            dev.render_frame()                      # before commit_world
        assert e.value.code == -2
        bad = di.Part(0, di.TRIS, verts=di.f32([(0, 0, 0), (1, 0, 0), (0, 1, 0)]),
                      idx=np.array([[0, 1, 7]], np.int32))
        dev.commit_part(bad)
        with pytest.raises(dpr.DprError) as e:
            dev.commit_world()                      # index validated on the GPU
        assert e.value.code == -1 and "index" in str(e.value)
        dev.clear_parts()
        hint = di.Part(0, di.SPHERES, spheres=di.f32([[0, 0, 0, 1]]))
        dev.commit_part(hint)
        dev.commit_world()
        b = dev.get_world_bounds()
        assert np.allclose(b, [-1, -1, -1, 1, 1, 1])
    finally:
        dev.release()


def test_consistency_error_on_every_rank():
    """Frame/Camera must be parameterised identically on all ranks; the
    collective render reports DPR_ERR_CONSISTENCY."""
    dpr = _dpr()
    sc = di.config1()
    devs = dpr.loopback_group(2, 0)
    try:
        for d in devs:
            d.commit_scene_parts(sc.parts)
            d.commit_world()
            d.set_camera(sc.camera)
        devs[0].set_frame(sc.frame)
        devs[1].set_frame(di.Frame(**{**sc.frame.__dict__, "spp": 2}))
        with pytest.raises(dpr.DprError) as e:
            dpr.render_frame_group(devs)
        assert e.value.code == -5
        devs[1].set_frame(sc.frame)
        dpr.render_frame_group(devs)
        assert devs[0].map_frame() is not None
        assert devs[1].map_frame() is None      # undefined on rank != 0, not an error
        assert devs[1].frame_ready()
        st = devs[1].get_stats()
        assert st["nranks"] == 2 and st["S"].shape == (3, 2, 2)
    finally:
        for d in devs:
            d.release()


def test_device_memory_parts_and_rebuild():
    """Parts committed from DEVICE memory (torch tensors) render identically to host parts;
    commit_world can be repeated (the bench step) with identical results."""
    import torch
    dpr = _dpr()
    sc = di.config2(nranks=1, G=31, W=64, H=64, spp=2, spp_batch=2)
    p = sc.parts[0]
    imgs = []
    for device_arrays in (False, True):
        dev = dpr.Device.create(0, 1, 0)
        try:
            if device_arrays:
                q = di.Part(**p.__dict__)
                q.verts = torch.from_numpy(p.verts).cuda()
                q.idx = torch.from_numpy(p.idx).cuda()
                dev.commit_part(q, device_arrays=True)
            else:
                dev.commit_part(p)
            dev.set_camera(sc.camera)
            dev.set_frame(sc.frame)
            for _ in range(2):
                dev.commit_world()
                dev.render_frame()
                imgs.append(dev.map_frame().cpu().numpy().copy())
        finally:
            dev.release()
    for im in imgs[1:]:
        assert np.allclose(im, imgs[0], atol=1e-6)
