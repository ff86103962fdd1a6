"""One rank of a multi-process render (launched by tests/test_gpu_multiproc.py, one process per
rank; env RANK, WORLD_SIZE, MASTER_ADDR, MASTER_PORT).

  python -m tests.mp_worker <transport> <case> <out.npz>
transport: hostcoll  -- torch.distributed gloo for the control collectives, ray records and the
                        a7 reduction through CUDA IPC peer memory; every rank on cuda:0
           nccl      -- the NCCL device (dpr_create_device), rank r on cuda:r
Rank 0 writes the frame, the P13 dumps and the routing statistics to out.npz."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def scene(case: str, nranks: int):
    import dpr_inputs as di
    if case == "c1":
        sc = di.config1()
        return sc.parts, sc.camera, sc.frame
    if case == "c2":
        sc = di.config2(nranks=nranks, G=41, W=64, H=48, spp=4, spp_batch=2)
        return sc.parts, sc.camera, sc.frame
    # random overlapping partition, depth 3, AO, bounces
    rng = np.random.default_rng(7)
    ntri, nsph = 300, 80
    c = rng.uniform(-1, 1, size=(ntri, 1, 3))
    v = (c + rng.uniform(-0.25, 0.25, size=(ntri, 3, 3))).astype(np.float32)
    sp = np.concatenate([rng.uniform(-1, 1, (nsph, 3)), rng.uniform(0.05, 0.2, (nsph, 1))], 1).astype(np.float32)
    tr, srk = rng.integers(0, nranks, ntri), rng.integers(0, nranks, nsph)
    parts = []
    for r in range(nranks):
        tv = v[tr == r].reshape(-1, 3)
        if tv.shape[0]:
            parts.append(di.Part(r, di.TRIS, albedo=(0.6, 0.5 + 0.03 * r, 0.4), verts=tv,
                                 idx=np.arange(tv.shape[0], dtype=np.int32).reshape(-1, 3)))
        s = sp[srk == r]
        if s.shape[0]:
            parts.append(di.Part(r, di.SPHERES, albedo=(0.3, 0.7, 0.2), spheres=s))
    cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, 40, 40)
    fr = di.Frame(W=40, H=40, spp=2, spp_batch=1, max_depth=3, ao_k=2, ao_radius=0.6,
                  light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3))
    return parts, cam, fr


def main():
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("DPR_MP_WATCHDOG_S", "240")), exit=True)
    transport, case, out = sys.argv[1], sys.argv[2], sys.argv[3]
    import torch
    import torch.distributed as dist
    import dpr_inputs as di
    from paper_2407_00179_b200 import dpr
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if transport == "hostcoll":
        dev = dpr.Device.create_hostcoll(0)
    else:
        dev = dpr.Device.create_distributed(rank)
    parts, cam, fr = scene(case, world)
    fr = di.Frame(**{**fr.__dict__, "flags": fr.flags | dpr.DPR_FLAG_DEBUG_DUMPS})
    try:
        dev.commit_scene_parts(parts)
        dev.commit_world()
        dev.set_camera(cam)
        dev.set_frame(fr)
        for i in range(2):  # the second frame reuses the IPC mappings / step graph
            dev.render_frame()
            print(f"rank {rank}: frame {i} ok", flush=True)
        st = dev.get_stats()
        ss = dev.get_step_stats()
        img = dev.map_frame()
        if rank == 0:
            e, o = dev.get_debug(fr.spp, fr.max_depth, fr.W * fr.H)
            np.savez(out, rgba=img.reshape(-1, 4).cpu().numpy().astype(np.float64),
                     events=e.cpu().numpy(), occl=o.cpu().numpy(), S=st["S"], V=st["V"],
                     rays=st["rays"], steps=st["steps"], step_S=ss["S"], step_V=ss["V"],
                     step_ms=ss["ms"], exch=st["exchanged_bytes_local"], loop=st["step_loop_device"])
        else:
            assert img is None
        torch.cuda.synchronize()
    except BaseException:
        import traceback
        traceback.print_exc()
        sys.stdout.flush()
        os._exit(1)  # the peers' pending collectives fail instead of waiting forever
    dev.release()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
