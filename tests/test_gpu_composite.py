"""NEXT row f3: the ANARI-Composite contrast device (P:534-647 S5.1) on the paper's E5 scene
(4^3 boxes pseudo-randomly interleaved across 4 ranks).  Parity: the GPU's
local renders + parallel direct send + per-pixel depth sort/over + gather equals the
oracle's per-rank local renders composited in numpy (oracle.deep_composite).  And the
paper's point: the composite misses the cross-rank shadows that ray forwarding produces."""
import numpy as np
import pytest

import dpr_inputs as di
import oracle as orc
from tests.gpu_helpers import MAX_ABS, MEAN_ABS, assert_pixels_close, gpu_render

pytestmark = pytest.mark.gpu


def _oracle_composite(sc):
    frs = [orc.render_local_fragments(sc.parts, r, sc.camera, sc.frame) for r in range(sc.nranks)]
    return orc.deep_composite(np.stack([f[0] for f in frs]), np.stack([f[1] for f in frs]), sc.frame.B)


@pytest.mark.parametrize("nranks", [2, 4])
def test_composite_matches_oracle_and_misses_shadows(nranks):
    from paper_2407_00179_b200 import dpr
    sc = di.boxes_scene(nranks=nranks, W=96, H=80, spp=4)
    devs = dpr.loopback_group(nranks, 0)
    try:
        for d in devs:
            d.commit_scene_parts(sc.parts)
            d.commit_world()
            d.set_camera(sc.camera)
            d.set_frame(sc.frame)
        dpr.render_frame_composite_group(devs)
        comp = devs[0].map_frame().reshape(-1, 4).cpu().numpy().astype(np.float64)
        assert all(d.map_frame() is None for d in devs[1:])
    finally:
        for d in devs:
            d.release()
    ref = _oracle_composite(sc)
    assert_pixels_close(comp, ref)
    # ray forwarding (the method) vs compositing (the contrast): cross-rank shadows differ
    fwd = gpu_render(sc.parts, nranks, sc.camera, sc.frame, dumps=False)[0]
    diff = np.abs(fwd[:, :3] - comp[:, :3]).mean()
    assert diff > 20 * MEAN_ABS, diff


def test_composite_single_rank_equals_plain_render():
    """With one rank compositing is the identity: local render == the world render."""
    from paper_2407_00179_b200 import dpr
    sc = di.boxes_scene(nranks=1, W=64, H=64, spp=2)
    dev = dpr.Device.create(0, 1, 0)
    try:
        dev.commit_scene_parts(sc.parts)
        dev.commit_world()
        dev.set_camera(sc.camera)
        dev.set_frame(sc.frame)
        dev.render_frame_composite()
        comp = dev.map_frame().reshape(-1, 4).cpu().numpy().astype(np.float64)
        dev.render_frame()
        plain = dev.map_frame().reshape(-1, 4).cpu().numpy().astype(np.float64)
    finally:
        dev.release()
    assert_pixels_close(comp, plain)
