"""Compare the two kernel-timing methods and the two step loops on one workload:
CUDA events around the launches (host loop) vs globaltimer first-CTA .. last-CTA spans (both
loops), and the frame time of the host vs the device-driven step loop.
  python tools/timing_check.py [c1|c2|c3|c4] [frames] [nranks(loopback)]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import dpr_inputs as di  # noqa: E402
from bench import make_scene  # noqa: E402


def run(cfg, frames, loop, nranks):
    os.environ["DPR_STEP_LOOP"] = loop
    import torch
    from paper_2407_00179_b200 import dpr
    sc = make_scene(cfg, nranks)
    devs = [dpr.Device.create(0, 1, 0)] if nranks == 1 else dpr.loopback_group(nranks, 0)
    for d in devs:
        d.commit_scene_parts(sc.parts)
        d.commit_world()
        d.set_camera(sc.camera)
        d.set_frame(sc.frame)
    out = []
    for i in range(frames + 2):
        if nranks == 1:
            devs[0].render_frame()
        else:
            dpr.render_frame_group(devs)
        st = devs[0].get_stats()
        ss = devs[0].get_step_stats()
        if i >= 2:
            out.append({"ms_frame": st["ms_frame"], "ev_or_span_path": st["ms_trace_path"],
                        "ev_or_span_occl": st["ms_trace_occl"], "span_path": st["ms_kernel_span"][0],
                        "span_occl": st["ms_kernel_span"][1], "steps": st["steps"],
                        "step_ms": [round(x, 4) for x in ss["ms"]], "launches": st["kernel_launches_local"]})
    torch.cuda.synchronize()
    for d in devs:
        d.release()
    keys = [k for k in out[0] if k not in ("step_ms",)]
    res = {k: float(np.median([o[k] for o in out])) for k in keys}
    res["step_ms"] = out[-1]["step_ms"]
    return res


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    for loop in ("host", "device"):
        print(json.dumps({"config": cfg, "nranks": n, "loop": loop, **run(cfg, frames, loop, n)}), flush=True)
