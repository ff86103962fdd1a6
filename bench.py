#!/usr/bin/env python
"""Benchmark: rays/sec and ms/frame of the data-parallel wavefront ray tracer (BASELINE.json
metric) on BASELINE configs[1]: a ~10M-triangle gyroid mesh spatially partitioned over the N
ranks, 1024x1024, 16 spp, shadows + ambient occlusion (K=4, r=0.25, depth 1).

One step = one pass of the whole hot path: dpr_commit_world (GPU LBVH rebuild from the
resident parts, row a1) + dpr_render_frame (rows a2-a7: primary generation, trace, route,
shade/spawn, exchange, framebuffer reduce).  Timed with CUDA events on the library's stream,
barrier + synchronize on both sides, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  N>1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

--impl reference times the CPU oracle (oracle/, the definition the CUDA path is checked
against) on a bounded pixel sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import dpr_inputs as di  # noqa: E402

METRIC = "rays/sec and ms/frame (device-timed, max over ranks)"
WORKLOAD = ("configs[1]: synthetic ~10M-triangle gyroid (marching tetrahedra G=301) spatially "
            "partitioned over N ranks, 1024x1024, 16 spp, shadows+AO (K=4, r=0.25, depth 1)")
WORKLOADS = {
    "c1": "configs[0]: two-rank world of 4 spheres + ground plane split by x-half, 64x64, 1 spp, AO 4, depth 2",
    "c2": WORKLOAD,
    "c3": "configs[2]: structured 1024^3 float32 volume split into per-rank bricks, DVR with volume "
          "shadows (1 spp, depth 1), 1920x1080",
    "c4": "configs[3]: 50M spheres in 1000 Gaussian clusters + ~5M-triangle gyroid, 1920x1080, 1 spp, depth 4",
    "c5": "configs[4]: ~100M-triangle gyroid + 1024^3 volume bricks, 3840x2160, 64 spp (batches of 4), depth 2",
}


def make_scene(cfg: str, world: int):
    if cfg == "c1":
        sc = di.config1()
        if world == 1:
            sc.parts = di.union_parts(sc.parts)
            sc.nranks = 1
        return sc
    if cfg == "c3":
        return di.config3(nranks=world)
    if cfg == "c4":
        return di.config4(nranks=world)
    if cfg == "c5":
        return di.config5(nranks=world)
    # one 16-spp batch on one GPU; 2 batches of 8 spp when the world is split (bounds the
    # per-peer send queues: worst case every ray of a batch goes to one peer)
    return di.config2(nranks=world, spp_batch=16 if world == 1 else 8)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profile_traffic():
    """dram bytes per launch from the committed ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        loaded = [x for x in sm if x > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------------------
PHASES = ("build", "gen", "trace_path", "trace_occl", "exchange", "reduce")


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(scene, seconds: float = 12.0):
    """Time the oracle (as it stands) on a random pixel subset of the workload, all samples
    of each pixel (paths are independent under Philox, so a subset is an exact sample)."""
    import oracle as orc
    t0 = time.time()
    parts = di.union_parts(scene.parts)
    osc = orc.OracleScene(parts, 1)
    t_build = time.time() - t0
    P = scene.frame.W * scene.frame.H
    rng = np.random.default_rng(1)
    n = 64
    while True:
        pix = np.sort(rng.choice(P, size=n, replace=False))
        t1 = time.time()
        r = orc.render(osc, scene.camera, scene.frame, pixels=pix, dp=False, dumps=False)
        dt = time.time() - t1
        if dt >= seconds or n >= P:
            break
        n = int(min(P, max(2 * n, n * seconds / max(dt, 1e-3) * 1.1)))
    rays = int(r.gen.sum())
    return {"value": rays / dt, "unit": "rays/s", "cores": os.cpu_count(), "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{n} random pixels x {scene.frame.spp} spp of the workload ({rays} rays) in "
                      f"{dt:.1f} s; oracle BVH build over {osc.nprims} prims {t_build:.1f} s not included",
            "seconds": dt}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    scene = make_scene(args.config, 1)
    if args.flags:
        scene.frame = di.Frame(**{**scene.frame.__dict__, "flags": scene.frame.flags | args.flags})
    import oracle as orc
    parts = di.union_parts(scene.parts)
    osc = orc.OracleScene(parts, 1)
    P = scene.frame.W * scene.frame.H
    rng = np.random.default_rng(2)
    npix = min(P, int(os.environ.get("DPR_REF_PIXELS", {"c1": 4096, "c3": 2048}.get(args.config, 8192))))
    times, rays = [], []
    for i in range(args.warmup + args.steps):
        pix = np.sort(rng.choice(P, size=npix, replace=False))
        t0 = time.time()
        r = orc.render(osc, scene.camera, scene.frame, pixels=pix, dp=False, dumps=False)
        dt = time.time() - t0
        if i >= args.warmup:
            times.append(dt)
            rays.append(int(r.gen.sum()))
    value = sum(rays) / sum(times)
    frame_rays_est = np.mean(rays) * P / npix
    line = {"metric": METRIC, "value": value, "unit": "rays/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * float(np.mean(times)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config],
                       "step": f"oracle on {npix} random pixels x {scene.frame.spp} spp",
                       "frame_flags": int(scene.frame.flags),
                       "est_ms_per_full_frame": 1000 * frame_rays_est / value},
            "cpu_baseline": {"value": value, "unit": "rays/s", "cores": os.cpu_count(),
                             "kind": "oracle",
                             "sample": f"{npix} random pixels x {scene.frame.spp} spp per step"},
            "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------
SMS, SCHED_PER_SM = 148, 4  # B200: 148 SMs x 4 warp schedulers, one warp-instruction issue / cycle each


def kernel_roofline(args, acc, ms_per_step, clocks):
    """The dominant trace kernel against the roof that binds it.

    Its duration is measured live (per-launch average: CUDA events on the library stream in
    host loops, globaltimer first-CTA-start .. last-CTA-end stamps inside the device-driven
    loop's graph, where events cannot be recorded).  Three fractions:
      touched: SURVEY 8(d) algorithmic bytes (records + 80 B/wide-node visit + 48 B/triangle
               + 16 B/sphere + 32 B/volume sample, exact device counters) / time vs HBM --
               most of these bytes hit L1/L2 (the node hierarchy is L2-resident);
      dram:    ncu dram__bytes_read+write per launch (profiles/traffic.json) / time vs HBM;
      issue:   ncu smsp__inst_executed per launch / time vs 148 SMs x 4 schedulers x the SM
               clock sampled during the run -- the roof the kernel actually presses on.
    "bound" names the largest fraction's roof."""
    peak, peak_src = measured_peaks()
    if acc["ms_path"] >= acc["ms_occl"]:
        kname, ms, n, b = "k_trace_path", acc["ms_path"], acc["n_path"], acc["b_path"]
    else:
        kname, ms, n, b = "k_trace_occl", acc["ms_occl"], acc["n_occl"], acc["b_occl"]
    avg_s = ms / max(n, 1) / 1000.0
    bytes_per_launch = b / max(n, 1)
    touched = bytes_per_launch / avg_s / 1e9 if avg_s > 0 else 0.0
    tkey = args.config + (f"+f{args.flags}" if args.flags else "") + ("" if args.mode == "dp" else f"+{args.mode}")
    tr = (profile_traffic() or {}).get(tkey, {}).get(kname, {})
    traffic = tr.get("dram_bytes_per_launch")
    clk_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    issue_peak = SMS * SCHED_PER_SM * clk_mhz * 1e6 / 1e9  # G warp-instructions / s
    inst = tr.get("inst_executed_per_launch")
    fr = {"touched": touched / peak}
    out = {"kernel": kname, "avg_launch_ms": avg_s * 1000, "launches_per_step": n / max(args.steps, 1),
           "share_of_step": (ms / args.steps) / ms_per_step,
           "other_kernel_ms_per_step": ((acc["ms_occl"] if kname == "k_trace_path" else acc["ms_path"]) / args.steps),
           "touched": {"bytes_per_launch": bytes_per_launch, "achieved_gbs": touched, "peak_gbs": peak,
                       "frac": touched / peak},
           "traffic": traffic, "peak_source": peak_src, "ncu_source": tr.get("source")}
    if traffic:
        dram = traffic / avg_s / 1e9
        fr["dram"] = dram / peak
        out["dram"] = {"bytes_per_launch": traffic, "achieved_gbs": dram, "peak_gbs": peak, "frac": dram / peak}
    if inst:
        ach = inst / avg_s / 1e9
        fr["issue"] = ach / issue_peak
        out["issue"] = {"warp_inst_per_launch": inst, "achieved_ginst_s": ach, "peak_ginst_s": issue_peak,
                        "frac": ach / issue_peak, "sm_mhz": clk_mhz,
                        "ncu_issue_active_pct": tr.get("issue_active_pct")}
    if tr.get("active_threads_per_warp_inst") is not None:
        out["simt_efficiency"] = tr["active_threads_per_warp_inst"] / 32.0
        out["warps_active_pct"] = tr.get("warps_active_pct")
    if "issue" in fr and fr["issue"] >= fr.get("dram", 0):
        out.update(bound="issue", achieved=out["issue"]["achieved_ginst_s"], peak=issue_peak,
                   unit="Gwarp-inst/s", frac=fr["issue"])
    elif "dram" in fr:
        out.update(bound="hbm", achieved=out["dram"]["achieved_gbs"], peak=peak, unit="GB/s", frac=fr["dram"])
    else:  # no ncu capture of this workload committed: the touched-bytes roof
        out.update(bound="hbm-touched", achieved=touched, peak=peak, unit="GB/s", frac=fr["touched"])
    out["touched_frac"] = fr["touched"]
    out["dram_frac"] = fr.get("dram")
    out["issue_frac"] = fr.get("issue")
    return out


def step_report(dev, world, ms_per_step):
    """Per-step routing of the last frame (P8b): steps, per-step latency, exchanged bytes per
    step (rays forwarded / spawned across ranks x record size) and the busiest pair."""
    ss = dev.get_step_stats()
    S = ss["S"]
    if not len(S):
        return None
    rec = np.array([64, 48, 48], np.int64)
    off = S.copy()
    for r in range(S.shape[2]):
        off[:, :, r, r] = 0
    bytes_pair = (off * rec[None, :, None, None]).sum(axis=1)  # [step][src][dst]
    out_rank = bytes_pair.sum(axis=2)                          # [step][src]
    in_rank = bytes_pair.sum(axis=1)                           # [step][dst]
    ms = ss["ms"]
    busiest = bytes_pair.reshape(len(S), -1).max(axis=1)
    per_step_max = np.maximum(out_rank.max(axis=1), in_rank.max(axis=1))
    rate = [float(b / (t * 1e-3) / 1e9) if t > 0 else None for b, t in zip(per_step_max, ms)]
    return {"n": int(ss["nsteps"]), "ms": [round(float(x), 4) for x in ms],
            "sync_ms": [round(float(x), 4) for x in ss["sync_ms"]],
            "exchange_bytes_max_rank": [int(x) for x in per_step_max],
            "busiest_pair_bytes": [int(x) for x in busiest],
            "exchange_gbs_per_rank_lower_bound": rate,
            "nvlink_gbs_per_direction": 900.0,
            "note": "fused exchange: records are written into peers' queues by the shading / resolve "
                    "kernels, overlapping the step's compute; the rate is bytes of the busiest rank / "
                    "whole step time (a lower bound of the link rate)"}


def parity_check(dev, scene, rank, world, npix=600):
    """After the timed region: one frame with the P13 dumps; rank 0 checks sampled pixels bit-exact
    (events, occlusion bits) and within the north_star tolerance against the oracle's routing
    simulator over the same partitioned world (tests/ hold the full parity suite)."""
    fr = di.Frame(**{**scene.frame.__dict__, "flags": scene.frame.flags | 2})
    dev.set_frame(fr)
    dev.commit_world()
    dev.render_frame()
    res = None
    if rank == 0:
        import oracle as orc
        e, o = dev.get_debug(fr.spp, fr.max_depth, fr.W * fr.H)
        img = dev.map_frame().reshape(-1, 4).cpu().numpy().astype(np.float64)
        P = fr.W * fr.H
        pix = np.sort(np.random.default_rng(9).choice(P, size=min(npix, P), replace=False))
        ora = orc.render(orc.OracleScene(scene.parts, world), scene.camera, fr, pixels=pix, dp=True)
        ev = e.cpu().numpy()[:, :, pix]
        oc = o.cpu().numpy()[:, :, pix]
        d = np.abs(img[pix] - ora.rgba)
        res = {"pixels": int(len(pix)), "events_bitexact": bool(np.array_equal(ev, ora.events)),
               "occl_bitexact": bool(np.array_equal(oc, ora.occl)),
               "max_abs": float(d.max()), "mean_abs_max_channel": float(d.mean(axis=0).max()),
               "within_tolerance": bool(d.max() <= 1e-3 and d.mean(axis=0).max() <= 1e-4)}
        res["ok"] = res["events_bitexact"] and res["occl_bitexact"] and res["within_tolerance"]
    dev.set_frame(scene.frame)
    return res


def run_gpu(args):
    import torch
    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # the communicator's rank count / transports (NVLS, P2P) in the log; ncclCommCount in the line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2407_00179_b200 import dpr
    scene = make_scene(args.config, 1 if args.mode == "replicated" else world)
    if args.flags:
        scene.frame = di.Frame(**{**scene.frame.__dict__, "flags": scene.frame.flags | args.flags})
    my_parts = [p for p in scene.parts if p.rank == rank or args.mode == "replicated"]
    if args.mode == "replicated":
        my_parts = [di.Part(**{**p.__dict__, "rank": rank}) for p in my_parts]

    def render():
        if args.mode == "replicated":
            dev.render_frame_replicated()
        elif args.mode == "composite":
            dev.render_frame_composite()
        else:
            dev.render_frame()
    if world > 1:
        dev = dpr.Device.create_distributed(local)
    else:
        dev = dpr.Device.create(0, 1, local)
    for p in my_parts:
        dev.commit_part(p)
    dev.commit_world()
    dev.set_camera(scene.camera)
    dev.set_frame(scene.frame)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident step: LBVH rebuild + collective render -----------------------
    for _ in range(args.warmup):
        dev.commit_world()
        render()
    barrier()
    acc = {"rays": 0, "launches": 0, "ms_path": 0.0, "n_path": 0, "ms_occl": 0.0, "n_occl": 0,
           "b_path": 0, "b_occl": 0, "ms_frame": [], "ms_build": [], "steps": 0, "exch": 0,
           "ms_exch": 0.0, "nodes": 0, "tris": 0}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        time.sleep(0.3)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            dev.commit_world()
            render()
            st = dev.get_stats()
            acc["rays"] += int(st["rays"].sum())
            acc["launches"] += st["kernel_launches_local"]
            acc["ms_path"] += st["ms_trace_path"]; acc["n_path"] += st["trace_path_launches"]
            acc["ms_occl"] += st["ms_trace_occl"]; acc["n_occl"] += st["trace_occl_launches"]
            acc["b_path"] += st["path_bytes_alg_local"]; acc["b_occl"] += st["occl_bytes_alg_local"]
            acc["ms_frame"].append(st["ms_frame_max"]); acc["ms_build"].append(st["ms_build"])
            acc["steps"] += st["steps"]; acc["exch"] += st["exchanged_bytes_local"]
            acc["ms_exch"] += st["ms_exchange"]
            acc["nodes"] += st["node_visits_local"]; acc["tris"] += st["tri_tests_local"]
            acc["visits"] = acc.get("visits", 0) + int(np.asarray(st["V"]).sum())
            for k in PHASES:
                acc[f"ph_{k}"] = acc.get(f"ph_{k}", 0.0) + st[f"ms_{k}"]
            for k in range(2):
                for f in ("rays", "nodes", "tris"):
                    acc.setdefault(f"k{k}_{f}", 0)
                    acc[f"k{k}_{f}"] += st[f"kernel_{f}_local"][k]
            acc["bvh_nodes"] = st["bvh_nodes_local"]; acc["bvh_levels"] = st["bvh_levels_local"]
            acc["comm_nranks"] = st["comm_nranks"]; acc["step_loop_device"] = st["step_loop_device"]
        e1.record(stream)
        barrier()
    elapsed_ms = max_over_ranks(e0.elapsed_time(e1))
    clocks = clk.summary()
    rays_per_frame = acc["rays"] / args.steps  # global (stats are gathered over ranks)
    value = rays_per_frame * args.steps / (elapsed_ms / 1000.0)
    ms_per_step = elapsed_ms / args.steps

    # roofline of the dominant kernel (rank 0's launches; DESIGN.md section 7 "Roofline")
    roofline = kernel_roofline(args, acc, ms_per_step, clocks)

    steps_detail = step_report(dev, world, ms_per_step)

    # ---- e2e: through the public API from pinned HOST buffers ---------------------------
    pinned = []
    h2d = 0
    for p in my_parts:
        q = di.Part(**p.__dict__)
        def pin(a, dtype):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype)).pin_memory()
            return t.numpy(), t.numel() * t.element_size()
        if p.kind == di.TRIS:
            (q.verts, b0), (q.idx, b1) = pin(p.verts, np.float32), pin(p.idx, np.int32)
            h2d += b0 + b1
        elif p.kind == di.SPHERES:
            q.spheres, b0 = pin(p.spheres, np.float32)
            h2d += b0
        else:
            (q.voxels, b0), (q.tf, b1) = pin(p.voxels, np.float32), pin(p.tf, np.float32)
            h2d += b0 + b1
        pinned.append(q)
    fb_host = torch.empty((scene.frame.H, scene.frame.W, 4), dtype=torch.float32).pin_memory()
    d2h = fb_host.numel() * 4 if rank == 0 else 0

    def commit_inputs():
        dev.clear_parts()
        for q in pinned:
            dev.commit_part(q, async_copy=True)

    copy_stream = torch.cuda.Stream()
    copy_done = [None]

    def e2e_step():
        # software pipeline, one step = upload + build + render + readback: the NEXT step's
        # mesh upload (pinned host -> device on the library's copy stream) is issued first and
        # overlaps this step's render (the built world no longer needs the parts); the frame
        # is read back to pinned host memory on a side stream, overlapping the next LBVH
        # build (the next render waits for that copy before it rewrites the frame); commit_world
        # waits for the upload and rebuilds the LBVH for the next step
        commit_inputs()
        if copy_done[0] is not None:
            stream.wait_event(copy_done[0])
        render()
        img = dev.map_frame()
        if img is not None:
            ev = torch.cuda.Event()
            ev.record(stream)
            copy_stream.wait_event(ev)
            with torch.cuda.stream(copy_stream):
                fb_host.copy_(img, non_blocking=True)
            copy_done[0] = torch.cuda.Event()
            copy_done[0].record(copy_stream)
        dev.commit_world()

    def e2e_drain():
        # the last readback is inside the timed region
        if copy_done[0] is not None:
            stream.wait_event(copy_done[0])

    if not args.no_e2e:
        commit_inputs()
        dev.commit_world()
        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        e2e_drain()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e2e_drain()
        e1.record(stream)
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    else:
        e2e_ms = float("nan")
    e2e_value = rays_per_frame * args.steps / (e2e_ms / 1000.0)
    parity = None
    if world > 1 and not args.no_parity and args.mode == "dp":
        parity = parity_check(dev, scene, rank, world)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = oracle_sample(scene, seconds=args.cpu_seconds)
        line = {
            "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "resolution": [scene.frame.W, scene.frame.H],
                       "spp": scene.frame.spp, "spp_batch": scene.frame.spp_batch,
                       "triangles": scene.meta.get("ntris", sum(p.nprims() for p in scene.parts)), "parallelism": f"dp{world} (world partitioned, ray forwarding)",
                       "l2": "inputs larger than L2 (BVH+prims ~1.1 GB, ray queues ~5 GB per step)",
                       "step": "dpr_commit_world (LBVH rebuild) + dpr_render_frame",
                       "mode": args.mode, "frame_flags": int(scene.frame.flags)},
            "ms_per_frame": float(np.median(acc["ms_frame"])),
            "ms_per_frame_min_max": [float(np.min(acc["ms_frame"])), float(np.max(acc["ms_frame"]))],
            "ms_per_phase_rank0": {k: acc[f"ph_{k}"] / args.steps for k in PHASES},
            "ray_visits_per_s": acc["visits"] / (elapsed_ms / 1000.0),
            "ms_build": float(np.median(acc["ms_build"])),
            "rays_per_frame": rays_per_frame,
            "wavefront_steps_per_frame": acc["steps"] / args.steps,
            "exchange_bytes_per_frame_rank0": acc["exch"] / args.steps,
            "ms_exchange_per_frame_rank0": acc["ms_exch"] / args.steps,
            "work_rank0": {kn: {"rays_per_frame": acc[f"k{k}_rays"] / args.steps,
                                "nodes_per_ray": acc[f"k{k}_nodes"] / max(acc[f"k{k}_rays"], 1),
                                "tris_per_ray": acc[f"k{k}_tris"] / max(acc[f"k{k}_rays"], 1)}
                           for k, kn in enumerate(["k_trace_path", "k_trace_occl"])},
            "bvh": {"wide_nodes": acc["bvh_nodes"], "collapse_levels": acc["bvh_levels"]},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "rays/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps},
            "gpu_launches": int(acc["launches"]),
            "clocks": clocks,
            "step_loop": "device (CUDA graph per spp batch)" if acc.get("step_loop_device") else "host",
            "wavefront_steps": steps_detail,
        }
        if world > 1:
            line["nccl"] = {"comm_nranks": int(acc.get("comm_nranks", 0)),
                            "comm_nranks_ok": int(acc.get("comm_nranks", 0)) == world,
                            "exchange": os.environ.get("DPR_EXCHANGE", "fused")}
            line["parity"] = parity
        print(json.dumps(line), flush=True)
    dev.release()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dpr", choices=["dpr", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--flags", type=int, default=0,
                    help="extra frame flags: 8 = ring schedule (R-RING), 16 = delta tracking (R-DELTA)")
    ap.add_argument("--mode", default="dp", choices=["dp", "replicated", "composite"],
                    help="dp = ray forwarding over a partitioned world (the method, default); "
                         "replicated = whole world on every rank, pixels split (Barney mode, "
                         "P:663-668); composite = local renders + deep compositing (P:534-647)")
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="workload (default c2 = BASELINE configs[1], the metric's workload)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling)")
    ap.add_argument("--no-parity", action="store_true", help="skip the N>1 sampled parity check")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
