"""Helpers shared by the -m gpu parity tests: run a scene through the C ABI (the product
path) and through the oracle, and compare them."""
from __future__ import annotations

import numpy as np

import dpr_inputs as di

# pixel tolerances from BASELINE.json north_star ("max-abs 1e-3 and mean-abs 1e-4 per channel")
MAX_ABS = 1e-3
MEAN_ABS = 1e-4


def gpu_render(parts, nranks, cam, fr, dumps=True, loopback=True, frames=1):
    """Render through libdpr.  nranks > 1 uses the loopback group (N virtual ranks on one
    GPU, same kernels, exchange by device copies).  Returns (rgba[H*W,4], events, occl,
    stats) on host."""
    import torch
    from paper_2407_00179_b200 import dpr
    fr = di.Frame(**{**fr.__dict__, "flags": fr.flags | (dpr.DPR_FLAG_DEBUG_DUMPS if dumps else 0)})
    if nranks == 1:
        devs = [dpr.Device.create(0, 1, 0)]
    else:
        devs = dpr.loopback_group(nranks, 0)
    try:
        for d in devs:
            d.commit_scene_parts(parts)
            d.commit_world()
            d.set_camera(cam)
            d.set_frame(fr)
        for _ in range(frames):
            if nranks == 1:
                devs[0].render_frame()
            else:
                dpr.render_frame_group(devs)
        img = devs[0].map_frame()
        rgba = img.reshape(-1, 4).cpu().numpy().astype(np.float64)
        ev = oc = None
        if dumps:
            e, o = devs[0].get_debug(fr.spp, fr.max_depth, fr.W * fr.H)
            ev, oc = e.cpu().numpy(), o.cpu().numpy()
        stats = devs[0].get_stats()
        stats["step"] = devs[0].get_step_stats()
        others = [d.map_frame() for d in devs[1:]]
        assert all(o is None for o in others)
        torch.cuda.synchronize()
        return rgba, ev, oc, stats
    finally:
        for d in devs:
            d.release()


def oracle_render(parts, nranks, cam, fr, pixels=None, dp=True):
    import oracle as orc
    sc = orc.OracleScene(parts, nranks)
    return orc.render(sc, cam, fr, pixels=pixels, dp=dp, step_matrices=dp)


def assert_pixels_close(gpu_rgba, ora_rgba, max_abs=MAX_ABS, mean_abs=MEAN_ABS):
    d = np.abs(gpu_rgba - ora_rgba)
    assert d.max() <= max_abs, f"max-abs {d.max():.3g} > {max_abs}"
    m = d.mean(axis=0)
    assert (m <= mean_abs).all(), f"mean-abs per channel {m} > {mean_abs}"


def assert_parity(gpu, ora, check_routing=True):
    rgba, ev, oc, st = gpu
    assert np.array_equal(ev, ora.events), f"events differ at {np.argwhere(ev != ora.events)[:5]}"
    assert np.array_equal(oc, ora.occl), f"occl differ at {np.argwhere(oc != ora.occl)[:5]}"
    assert np.array_equal(st["rays"], ora.gen), (st["rays"], ora.gen)
    if check_routing and ora.S is not None:
        assert np.array_equal(st["S"], ora.S), (st["S"], ora.S)
        assert np.array_equal(st["V"], ora.V), (st["V"], ora.V)
        assert st["steps"] == int(ora.steps.sum()), (st["steps"], ora.steps)
        if ora.S_step is not None and "step" in st and len(ora.S_step) <= 256:
            # P8b per-step routing matrices and visits, bit-exact
            assert np.array_equal(st["step"]["S"], ora.S_step), "per-step S differ"
            assert np.array_equal(st["step"]["V"], ora.V_step), "per-step V differ"
    assert_pixels_close(rgba, ora.rgba)
