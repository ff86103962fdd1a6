"""Per-step routing and load balance (P:225-236 lock-step cost "limited by
the pair of ranks with the highest ray count"; P:1347-1366 partitioning).

configs[1]'s ~10M-triangle gyroid at 512x512, 4 spp (one batch) over N = 2, 4, 8 loopback ranks
(the same kernels as N GPUs, one GPU) for each partition strategy; per wavefront step the GPU's
routing matrix S_k and visits V_k (dpr_get_step_stats) are checked bit-exact against the
oracle's routing simulator (whole frame), then summarised:
  max/mean visits per rank over the frame (trace-work imbalance),
  per step: busiest rank (visits), busiest pair (rays), exchanged bytes,
  lock-step critical path = sum over steps of max_rank V_k[r] vs the balanced sum_k mean_r V_k[r]
  (in ray visits: every rank waits for the slowest at every step boundary).
One JSON line per (N, partition) -> profiles/r02_load_balance.jsonl
    python tools/load_balance_study.py [out.jsonl]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dpr_inputs as di  # noqa: E402

RES = int(os.environ.get("LB_RES", "512"))
SPP = int(os.environ.get("LB_SPP", "4"))
NS = [int(x) for x in os.environ.get("LB_N", "2,4,8").split(",")]


def main(out_path):
    import torch
    import oracle as orc
    from paper_2407_00179_b200 import dpr
    rec = np.array([64, 48, 48], np.int64)
    lines = []
    for N in NS:
        for strategy in di.PARTITIONS:
            sc = di.config2(nranks=N, W=RES, H=RES, spp=SPP, spp_batch=SPP, partition=strategy)
            devs = dpr.loopback_group(N, 0)
            try:
                for d in devs:
                    d.commit_scene_parts(sc.parts)
                    d.commit_world()
                    d.set_camera(sc.camera)
                    d.set_frame(sc.frame)
                dpr.render_frame_group(devs)
                torch.cuda.synchronize()
                st = devs[0].get_stats()
                ss = devs[0].get_step_stats()
            finally:
                for d in devs:
                    d.release()
            t0 = time.time()
            o = orc.render(orc.OracleScene(sc.parts, N), sc.camera, sc.frame, dp=True, dumps=False,
                           step_matrices=True)
            t_or = time.time() - t0
            S, V = ss["S"], ss["V"]
            exact = bool(np.array_equal(S, o.S_step) and np.array_equal(V, o.V_step) and
                         np.array_equal(st["S"], o.S) and np.array_equal(st["V"], o.V))
            vr = V.sum(axis=1)                     # [step][rank] visits, all kinds
            tot_r = vr.sum(axis=0)
            off = S.copy()
            for r in range(N):
                off[:, :, r, r] = 0
            pair_rays = off.sum(axis=1)            # [step][src][dst]
            pair_bytes = (off * rec[None, :, None, None]).sum(axis=1)
            crit = int(vr.max(axis=1).sum())
            bal = float(vr.mean(axis=1).sum())
            line = {"N": N, "partition": strategy, "resolution": RES, "spp": SPP, "triangles": sc.meta["ntris"],
                    "rays": int(st["rays"].sum()), "steps": int(len(S)),
                    "per_step_bitexact_vs_oracle": exact,
                    "visits_per_rank": tot_r.tolist(),
                    "visits_max_over_mean": float(tot_r.max() / tot_r.mean()),
                    "per_step_visits_max_rank": vr.max(axis=1).tolist(),
                    "per_step_busiest_pair_rays": pair_rays.reshape(len(S), -1).max(axis=1).tolist(),
                    "per_step_exchanged_bytes": pair_bytes.sum(axis=(1, 2)).tolist(),
                    "busiest_pair_rays_frame": int(pair_rays.sum(axis=0).max()),
                    "lockstep_critical_path_visits": crit, "balanced_visits": bal,
                    "lockstep_efficiency": bal / crit if crit else None,
                    "oracle_seconds": round(t_or, 1)}
            print(json.dumps(line), flush=True)
            lines.append(line)
    with open(out_path, "w") as f:
        for ln in lines:
            f.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "r02_load_balance.jsonl"))
