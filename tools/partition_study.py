"""NEXT row f2 measurement: how the partition strategy changes ray forwarding on configs[1]
(simple distributions "generally exchange more rays than with an optimized
partitioning", lock-step cost "limited by the pair of ranks with the highest ray count").
Loopback groups (N virtual ranks on one GPU, same kernels, fused exchange): per strategy and
N, rays generated, visits per ray, forwarded rays, busiest pair, steps, exchanged bytes, and
the single-GPU frame time (a proxy: all ranks share one GPU, so it measures total work, not
multi-GPU scaling).  One JSON line per (strategy, N).  PS_SCHEDULES=visit,ring adds the ring
schedule (NEXT row f4, DPR_FLAG_RING) for the same partitions."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dpr_inputs as di  # noqa: E402
from paper_2407_00179_b200 import dpr  # noqa: E402

G = int(os.environ.get("PS_G", "301"))
RES = int(os.environ.get("PS_RES", "512"))
SPP = int(os.environ.get("PS_SPP", "4"))
SCHEDULES = os.environ.get("PS_SCHEDULES", "visit").split(",")
STRATEGIES = os.environ.get("PS_STRATEGIES", ",".join(di.PARTITIONS)).split(",")
for N in (2, 4, 8):
    for strategy, schedule in [(a, b) for a in STRATEGIES for b in SCHEDULES]:
        sc = di.config2(nranks=N, G=G, W=RES, H=RES, spp=SPP, spp_batch=SPP, partition=strategy)
        if schedule == "ring":
            sc.frame = di.Frame(**{**sc.frame.__dict__, "flags": sc.frame.flags | dpr.DPR_FLAG_RING})
        devs = dpr.loopback_group(N, 0)
        try:
            for d in devs:
                d.commit_scene_parts(sc.parts)
                d.commit_world()
                d.set_camera(sc.camera)
                d.set_frame(sc.frame)
            dpr.render_frame_group(devs)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                dpr.render_frame_group(devs)
            e1.record()
            torch.cuda.synchronize()
            st = devs[0].get_stats()
            S, V = st["S"], st["V"]
            rays = int(st["rays"].sum())
            fwd = int(S.sum())
            pair = S.sum(axis=0)
            exch = sum(d.get_stats()["exchanged_bytes_local"] for d in devs)
            line = {"N": N, "partition": strategy, "schedule": schedule, "triangles": sc.meta["ntris"],
                    "resolution": RES, "spp": SPP, "rays": rays,
                    "visits_per_ray": float(V.sum() / rays), "forwarded_rays": fwd,
                    "forwarded_per_ray": fwd / rays, "busiest_pair_rays": int(pair.max()),
                    "steps": int(st["steps"]), "exchanged_bytes": int(exch),
                    "ms_per_frame_loopback_1gpu": e0.elapsed_time(e1) / 3}
            print(json.dumps(line), flush=True)
        finally:
            for d in devs:
                d.release()
