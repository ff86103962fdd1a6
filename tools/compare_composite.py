"""NEXT row f3 measurement: ray forwarding (the method) vs the compositing contrast device on
the paper's E5 scene (4^3 boxes over 4 ranks), 4 virtual ranks on ONE GPU
(loopback group; exchange by device copies) -- a single-GPU demonstration, not a multi-GPU
number.  Prints one JSON line: device ms per frame for both, and the image difference."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dpr_inputs as di  # noqa: E402
from paper_2407_00179_b200 import dpr  # noqa: E402


def main():
    W = H = int(os.environ.get("E5_RES", "1024"))
    spp = int(os.environ.get("E5_SPP", "16"))
    sc = di.boxes_scene(nranks=4, W=W, H=H, spp=spp)
    devs = dpr.loopback_group(4, 0)
    out = {"scene": f"E5 boxes 4^3 over 4 ranks, {W}x{H}, {spp} spp, AO 2, depth 2",
           "ranks": "4 virtual ranks on one B200 (loopback group)"}
    try:
        for d in devs:
            d.commit_scene_parts(sc.parts)
            d.commit_world()
            d.set_camera(sc.camera)
            d.set_frame(sc.frame)
        s = torch.cuda.current_stream()
        for name, fn in (("ray_forwarding", lambda: dpr.render_frame_group(devs)),
                         ("compositing", lambda: dpr.render_frame_composite_group(devs))):
            for _ in range(2):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(5):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            st = devs[0].get_stats()
            out[name] = {"ms_per_frame": e0.elapsed_time(e1) / 5, "rays_per_frame": int(st["rays"].sum()),
                         "wavefront_steps": int(st["steps"])}
            out[name + "_image"] = devs[0].map_frame().reshape(-1, 4).cpu().numpy().astype(np.float64)
        fwd, comp = out.pop("ray_forwarding_image"), out.pop("compositing_image")
        d = np.abs(fwd[:, :3] - comp[:, :3])
        out["image_difference"] = {"mean_abs": float(d.mean()), "max_abs": float(d.max()),
                                   "pixels_differing_gt_0.05": float((d.max(axis=1) > 0.05).mean())}
        out["note"] = ("compositing renders each rank's boxes with local shading only: shadows and AO "
                       "cast by other ranks' boxes are missing (P:645-647)")
    finally:
        for d in devs:
            d.release()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
