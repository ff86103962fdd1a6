"""One-off: configs[4] at full size on one GPU (100M-triangle gyroid + 1024^3 volume bricks,
3840x2160, 64 spp in batches of 4, depth 2): device frame time, and every event / occlusion
bit of a random pixel sample against the oracle."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dpr_inputs as di  # noqa: E402
import oracle as orc  # noqa: E402
from paper_2407_00179_b200 import dpr  # noqa: E402

t0 = time.time()
sc = di.config5(nranks=1)
print("scene", time.time() - t0, "s", sc.meta, flush=True)
fr = di.Frame(**{**sc.frame.__dict__, "flags": sc.frame.flags | dpr.DPR_FLAG_DEBUG_DUMPS})
dev = dpr.Device.create(0, 1, 0)
for p in sc.parts:
    dev.commit_part(p)
dev.commit_world()
dev.set_camera(sc.camera)
dev.set_frame(fr)
dev.render_frame()
torch.cuda.synchronize()
st = dev.get_stats()
rgba = dev.map_frame().reshape(-1, 4).cpu().numpy().astype(np.float64)
ev, oc = (x.cpu().numpy() for x in dev.get_debug(fr.spp, fr.max_depth, fr.W * fr.H))
res = {"ms_frame": st["ms_frame"], "ms_build": st["ms_build"], "rays": int(st["rays"].sum()),
       "rays_per_s": int(st["rays"].sum()) / (st["ms_frame"] / 1000.0)}
print(res, flush=True)
dev.release()
del dev
P = fr.W * fr.H
pix = np.sort(np.random.default_rng(9).choice(P, int(os.environ.get("C5_PIX", "150")), replace=False))
t0 = time.time()
osc = orc.OracleScene(sc.parts, 1)
tb = time.time() - t0
t0 = time.time()
o = orc.render(osc, sc.camera, fr, pixels=pix, dp=False)
to = time.time() - t0
ev_ok = bool(np.array_equal(ev[:, :, pix], o.events))
oc_ok = bool(np.array_equal(oc[:, :, pix], o.occl))
d = np.abs(rgba[pix] - o.rgba)
res.update({"pixels": int(pix.size), "events_equal": ev_ok, "occl_equal": oc_ok,
            "max_abs": float(d.max()), "mean_abs": float(d.mean()), "oracle_build_s": tb, "oracle_s": to,
            "volume_events": int(((o.events & 0x80000000) != 0).sum())})
print(json.dumps(res), flush=True)
