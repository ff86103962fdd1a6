"""NEXT row f4 (part): Barney's data-replicated mode -- every rank holds
the whole world, pixels are split by owner (p*N)/P, no ray forwarding; the frame equals the
single-world render bit-exactly in events / occlusion bits, pixels within tolerance."""
import numpy as np
import pytest

import dpr_inputs as di
from tests.gpu_helpers import assert_parity, oracle_render

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 3, 4])
def test_replicated_equals_union(n):
    from paper_2407_00179_b200 import dpr
    sc = di.config1()
    world = di.union_parts(sc.parts)
    fr = di.Frame(**{**sc.frame.__dict__, "flags": sc.frame.flags | dpr.DPR_FLAG_DEBUG_DUMPS})
    devs = dpr.loopback_group(n, 0) if n > 1 else [dpr.Device.create(0, 1, 0)]
    try:
        for d in devs:
            for p in world:            # the WHOLE world on every rank
                d.commit_part(p)
            d.commit_world()
            d.set_camera(sc.camera)
            d.set_frame(fr)
        if n > 1:
            dpr.render_frame_replicated_group(devs)
        else:
            devs[0].render_frame_replicated()
        rgba = devs[0].map_frame().reshape(-1, 4).cpu().numpy().astype(np.float64)
        ev, oc = devs[0].get_debug(fr.spp, fr.max_depth, fr.W * fr.H)
        st = devs[0].get_stats()
        g = (rgba, ev.cpu().numpy(), oc.cpu().numpy(), st)
    finally:
        for d in devs:
            d.release()
    o = oracle_render(world, 1, sc.camera, sc.frame, dp=False)
    assert_parity(g, o, check_routing=False)
