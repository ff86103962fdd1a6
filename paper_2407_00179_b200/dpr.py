"""Thin Python binding of libdpr.so (include/dpr.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module converts
dpr_inputs scene objects to the C structs, hands PyTorch's caching allocator and current
CUDA stream to the library (north_star: "PyTorch is used only for device memory, streams
and process groups"), and bootstraps the NCCL communicator through torch.distributed.
There is NO fallback: if the extension is missing or the GPU is absent, calls raise.
Names follow the C ABI (dpr_* without the prefix).
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DPR_LIB") or os.path.join(HERE, "libdpr.so")

DPR_OK = 0
DPR_MAX_RANKS = 16
DPR_FLAG_JITTER_CENTER = 1
DPR_FLAG_DEBUG_DUMPS = 2
DPR_FLAG_RING = 8
DPR_FLAG_DELTA = 16
# dpr_part_kind / dpr_memory (include/dpr.h)
DPR_PART_TRIANGLES, DPR_PART_SPHERES, DPR_PART_BRICK = 0, 1, 2
DPR_MEMORY_HOST, DPR_MEMORY_DEVICE, DPR_MEMORY_HOST_ASYNC = 0, 1, 2
ERRORS = {-1: "DPR_ERR_INVALID_ARG", -2: "DPR_ERR_STATE", -3: "DPR_ERR_CUDA", -4: "DPR_ERR_NCCL",
          -5: "DPR_ERR_CONSISTENCY", -6: "DPR_ERR_OOM", -7: "DPR_ERR_QUEUE_OVERFLOW"}


class DprError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


_c = ctypes
_P = _c.c_void_p


class dpr_part_desc(_c.Structure):
    _fields_ = [("kind", _c.c_int32), ("memory", _c.c_int32), ("albedo", _c.c_float * 3),
                ("n_verts", _c.c_int64), ("verts", _P), ("n_tris", _c.c_int64), ("idx", _P),
                ("n_spheres", _c.c_int64), ("spheres", _P), ("gdims", _c.c_int32 * 3),
                ("origin", _c.c_float * 3), ("spacing", _c.c_float * 3),
                ("cell_lo", _c.c_int32 * 3), ("cell_hi", _c.c_int32 * 3), ("voxels", _P),
                ("tf", _P), ("tf_lo", _c.c_float), ("tf_hi", _c.c_float),
                ("density_scale", _c.c_float), ("has_bounds_hint", _c.c_int32),
                ("bounds_hint", _c.c_float * 6)]


class dpr_camera_basis(_c.Structure):
    _fields_ = [("E", _c.c_float * 3), ("L", _c.c_float * 3), ("U", _c.c_float * 3),
                ("V", _c.c_float * 3), ("lens_radius", _c.c_float), ("focus_dist", _c.c_float)]


class dpr_frame_desc(_c.Structure):
    _fields_ = [("W", _c.c_int32), ("H", _c.c_int32), ("spp", _c.c_int32),
                ("spp_batch", _c.c_int32), ("max_depth", _c.c_int32), ("ao_k", _c.c_int32),
                ("ao_radius", _c.c_float), ("light_dir", _c.c_float * 3), ("E", _c.c_float * 3),
                ("A", _c.c_float * 3), ("B", _c.c_float * 3), ("dt", _c.c_float),
                ("seed", _c.c_uint64), ("flags", _c.c_uint32)]


R = DPR_MAX_RANKS


class dpr_stats(_c.Structure):
    _fields_ = [("nranks", _c.c_int32), ("rank", _c.c_int32),
                ("S", _c.c_int64 * (3 * R * R)), ("V", _c.c_int64 * (3 * R)),
                ("rays", _c.c_int64 * 3), ("steps", _c.c_int64),
                ("node_visits_local", _c.c_int64), ("tri_tests_local", _c.c_int64),
                ("sphere_tests_local", _c.c_int64), ("vol_samples_local", _c.c_int64),
                ("records_in_local", _c.c_int64), ("records_out_local", _c.c_int64),
                ("exchanged_bytes_local", _c.c_int64), ("kernel_launches_local", _c.c_int64),
                ("trace_path_launches", _c.c_int64), ("trace_occl_launches", _c.c_int64),
                ("ms_frame", _c.c_double), ("ms_build", _c.c_double), ("ms_gen", _c.c_double),
                ("ms_trace_path", _c.c_double), ("ms_trace_occl", _c.c_double),
                ("ms_exchange", _c.c_double), ("ms_reduce", _c.c_double),
                ("ms_frame_max", _c.c_double), ("path_bytes_alg_local", _c.c_int64),
                ("occl_bytes_alg_local", _c.c_int64), ("kernel_rays_local", _c.c_int64 * 2),
                ("kernel_nodes_local", _c.c_int64 * 2), ("kernel_tris_local", _c.c_int64 * 2),
                ("kernel_sphs_local", _c.c_int64 * 2), ("kernel_vols_local", _c.c_int64 * 2),
                ("bvh_nodes_local", _c.c_int64), ("bvh_levels_local", _c.c_int64),
                ("step_loop_device", _c.c_int64), ("graph_builds", _c.c_int64),
                ("comm_nranks", _c.c_int64), ("ms_kernel_span", _c.c_double * 2)]

    def to_dict(self) -> dict:
        n = self.nranks
        S = np.frombuffer(self.S, np.int64).reshape(3, R, R)[:, :n, :n].copy()
        V = np.frombuffer(self.V, np.int64).reshape(3, R)[:, :n].copy()
        arrays = ("S", "V", "rays", "kernel_rays_local", "kernel_nodes_local", "kernel_tris_local",
                  "kernel_sphs_local", "kernel_vols_local", "ms_kernel_span")
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in arrays}
        for k in arrays[3:]:
            d[k] = list(getattr(self, k))
        d.update(S=S, V=V, rays=np.frombuffer(self.rays, np.int64).copy())
        return d


ALLGATHER_FN = _c.CFUNCTYPE(_c.c_int, _P, _P, _P, _c.c_size_t)


class dpr_host_collectives(_c.Structure):
    _fields_ = [("allgather", ALLGATHER_FN), ("ctx", _P)]


ALLOC_FN = _c.CFUNCTYPE(_P, _P, _c.c_size_t, _P)
FREE_FN = _c.CFUNCTYPE(None, _P, _P, _c.c_size_t, _P)


class dpr_allocator(_c.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("ctx", _P)]


EXPORTS = ["dpr_get_unique_id", "dpr_create_device", "dpr_create_device_hostcoll", "dpr_create_loopback_group",
           "dpr_release_device", "dpr_commit_part", "dpr_clear_parts", "dpr_commit_world",
           "dpr_get_world_bounds", "dpr_set_camera", "dpr_set_frame", "dpr_render_frame",
           "dpr_render_frame_group", "dpr_render_frame_composite", "dpr_render_frame_composite_group",
           "dpr_render_frame_replicated", "dpr_render_frame_replicated_group",
           "dpr_frame_ready", "dpr_map_frame", "dpr_get_debug",
           "dpr_get_stats", "dpr_get_step_stats", "dpr_last_error", "dpr_exchange_plan",
           "dpr_test_step_barrier", "dpr_test_radix_sort"]

_lib = None


def load(path: str = LIB_PATH):
    """Load libdpr.so (must have been built; see paper_2407_00179_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libdpr.so not built ({path}); run __graft_entry__.build()")
    L = _c.CDLL(path)
    L.dpr_get_unique_id.argtypes = [_P]
    L.dpr_create_device.argtypes = [_c.c_int, _c.c_int, _c.c_int, _P, _P, _P, _P]
    L.dpr_create_loopback_group.argtypes = [_c.c_int, _c.c_int, _P, _P, _P]
    L.dpr_create_device_hostcoll.argtypes = [_c.c_int, _c.c_int, _c.c_int, _P, _P, _P, _P]
    L.dpr_get_step_stats.argtypes = [_P, _c.c_int, _P, _P, _P, _P, _P]
    L.dpr_test_step_barrier.argtypes = [_c.c_int, _c.c_int, _c.c_int, _P]
    L.dpr_test_radix_sort.argtypes = [_c.c_int, _P, _c.c_int64, _P]
    for n in ("dpr_release_device", "dpr_clear_parts", "dpr_commit_world", "dpr_render_frame",
              "dpr_render_frame_composite", "dpr_render_frame_replicated"):
        getattr(L, n).argtypes = [_P]
    L.dpr_render_frame_composite_group.argtypes = [_P, _c.c_int]
    L.dpr_render_frame_replicated_group.argtypes = [_P, _c.c_int]
    L.dpr_commit_part.argtypes = [_P, _P]
    L.dpr_get_world_bounds.argtypes = [_P, _P]
    L.dpr_set_camera.argtypes = [_P, _P]
    L.dpr_set_frame.argtypes = [_P, _P]
    L.dpr_render_frame_group.argtypes = [_P, _c.c_int]
    L.dpr_frame_ready.argtypes = [_P, _c.c_int]
    L.dpr_map_frame.argtypes = [_P, _P, _P, _P, _P]
    L.dpr_get_debug.argtypes = [_P, _P, _P]
    L.dpr_get_stats.argtypes = [_P, _P]
    L.dpr_last_error.argtypes = [_P]
    L.dpr_last_error.restype = _c.c_char_p
    L.dpr_exchange_plan.argtypes = [_c.c_int, _c.c_int, _P, _c.c_int64, _P, _P, _P]
    for n in EXPORTS:
        if n != "dpr_last_error":
            getattr(L, n).restype = _c.c_int
    _lib = L
    return L


def _check(rc: int, dev=None):
    if rc < 0:
        msg = load().dpr_last_error(dev).decode()
        raise DprError(rc, msg)
    return rc


def exchange_plan(nranks: int, rank: int, counts: np.ndarray, capacity: int):
    """dpr_exchange_plan: host-only planner of the next input queue layout."""
    c = np.ascontiguousarray(counts, np.int64).reshape(nranks * nranks)
    off = np.zeros(nranks, np.int64)
    tin, gt = _c.c_int64(0), _c.c_int64(0)
    rc = load().dpr_exchange_plan(nranks, rank, c.ctypes.data, capacity, off.ctypes.data,
                                  _c.byref(tin), _c.byref(gt))
    return rc, off, tin.value, gt.value


def test_step_barrier(cuda_device: int, nranks: int, iters: int) -> int:
    """dpr_test_step_barrier: mismatching boundaries of the emulated mailbox barrier."""
    m = _c.c_int64(-1)
    _check(load().dpr_test_step_barrier(cuda_device, nranks, iters, _c.byref(m)))
    return m.value


def test_radix_sort(cuda_device: int, keys_ptr: int, n: int, perm_ptr: int) -> None:
    """dpr_test_radix_sort: the build's stable LSD key sort; keys / perm are device pointers."""
    _check(load().dpr_test_radix_sort(cuda_device, keys_ptr, n, perm_ptr))


def get_unique_id() -> bytes:
    buf = (_c.c_uint8 * 128)()
    _check(load().dpr_get_unique_id(buf))
    return bytes(buf)


# ----------------------------------------------------------------------------------------
class _CudaArray:
    """Zero-copy view of library-owned device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class TorchAllocator:
    """dpr_allocator backed by torch's caching allocator on the current device/stream."""

    def __init__(self, device: int):
        import torch
        self.torch = torch
        self.device = device

        def _alloc(ctx, nbytes, stream):
            try:
                return self.torch.cuda.caching_allocator_alloc(int(nbytes), self.device, stream)
            except Exception:
                return None

        def _free(ctx, ptr, nbytes, stream):
            if ptr:
                self.torch.cuda.caching_allocator_delete(ptr)

        self._a = ALLOC_FN(_alloc)
        self._f = FREE_FN(_free)
        self.struct = dpr_allocator(self._a, self._f, None)


def part_desc(p, keep: list, device_arrays: bool = False, async_copy: bool = False) -> dpr_part_desc:
    """A part object (kind, albedo, verts/idx | spheres | brick fields, as dpr_inputs.Part;
    numpy host arrays or torch CUDA tensors) -> dpr_part_desc.
    async_copy: DPR_MEMORY_HOST_ASYNC (pinned host arrays, read until dpr_commit_world)."""
    s = dpr_part_desc()
    s.kind = p.kind
    s.memory = (DPR_MEMORY_DEVICE if device_arrays else
                DPR_MEMORY_HOST_ASYNC if async_copy and p.kind != DPR_PART_BRICK else DPR_MEMORY_HOST)
    s.albedo = (_c.c_float * 3)(*[float(x) for x in p.albedo])

    def ptr(a, dtype):
        if a is None:
            return None
        if device_arrays:
            keep.append(a)
            return a.data_ptr()
        a = np.ascontiguousarray(a, dtype)
        keep.append(a)
        return a.ctypes.data

    if p.kind == DPR_PART_TRIANGLES:
        s.n_verts, s.verts = int(p.verts.shape[0]), ptr(p.verts, np.float32)
        s.n_tris, s.idx = int(p.idx.shape[0]), ptr(p.idx, np.int32)
    elif p.kind == DPR_PART_SPHERES:
        s.n_spheres, s.spheres = int(p.spheres.shape[0]), ptr(p.spheres, np.float32)
    else:
        s.gdims = (_c.c_int32 * 3)(*p.gdims)
        s.origin = (_c.c_float * 3)(*p.origin)
        s.spacing = (_c.c_float * 3)(*p.spacing)
        s.cell_lo = (_c.c_int32 * 3)(*p.cell_lo)
        s.cell_hi = (_c.c_int32 * 3)(*p.cell_hi)
        s.voxels, s.tf = ptr(p.voxels, np.float32), ptr(p.tf, np.float32)
        s.tf_lo, s.tf_hi, s.density_scale = p.tf_lo, p.tf_hi, p.density_scale
    return s


def camera_struct(cam) -> dpr_camera_basis:
    c = dpr_camera_basis()
    c.E, c.L, c.U, c.V = [(_c.c_float * 3)(*[float(x) for x in v]) for v in (cam.E, cam.L, cam.U, cam.V)]
    c.lens_radius, c.focus_dist = float(getattr(cam, "lens_radius", 0.0)), float(getattr(cam, "focus_dist", 0.0))
    return c


def frame_struct(f) -> dpr_frame_desc:
    o = dpr_frame_desc()
    o.W, o.H, o.spp, o.spp_batch, o.max_depth, o.ao_k = f.W, f.H, f.spp, f.spp_batch, f.max_depth, f.ao_k
    o.ao_radius = f.ao_radius
    o.light_dir, o.E, o.A, o.B = [(_c.c_float * 3)(*[float(x) for x in v])
                                  for v in (f.light_dir, f.E, f.A, f.B)]
    o.dt, o.seed, o.flags = f.dt, f.seed, f.flags
    return o


class Device:
    """One rank's dpr_device.  Use Device.create(...) (collective) or loopback_group(...)."""

    def __init__(self, handle, rank: int, nranks: int, alloc: Optional[TorchAllocator],
                 stream_obj=None):
        self.h = _P(handle)
        self.rank = rank
        self.nranks = nranks
        self._alloc = alloc
        self._stream = stream_obj
        self._keep: list = []

    # -- lifetime -----------------------------------------------------------------------
    @classmethod
    def create(cls, rank: int = 0, nranks: int = 1, cuda_device: int = 0, uid: Optional[bytes] = None,
               stream=None, torch_alloc: bool = True) -> "Device":
        import torch
        torch.cuda.set_device(cuda_device)
        stream = stream or torch.cuda.current_stream(cuda_device)
        alloc = TorchAllocator(cuda_device) if torch_alloc else None
        h = _P()
        ub = (_c.c_uint8 * 128).from_buffer_copy(uid) if uid else None
        _check(load().dpr_create_device(rank, nranks, cuda_device, ub, _P(stream.cuda_stream),
                                        _c.byref(alloc.struct) if alloc else None, _c.byref(h)))
        return cls(h.value, rank, nranks, alloc, stream)

    @classmethod
    def create_distributed(cls, cuda_device: int, stream=None) -> "Device":
        """Collective creation over an initialised torch.distributed group: rank 0 makes the
        NCCL unique id and broadcasts it (P:460-461 collaborative device creation)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [get_unique_id() if rank == 0 and world > 1 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        return cls.create(rank, world, cuda_device, obj[0], stream)

    @classmethod
    def create_hostcoll(cls, cuda_device: int = 0, group=None, stream=None) -> "Device":
        """dpr_create_device_hostcoll over a torch.distributed (e.g. gloo) group: the control
        collectives are torch all-gathers of byte tensors, the ray records move through CUDA
        IPC peer memory (processes may share one GPU)."""
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(cuda_device)
        stream = stream or torch.cuda.current_stream(cuda_device)
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def _allgather(ctx, send, recv, nbytes):
            try:
                src = torch.frombuffer(bytearray(_c.string_at(send, nbytes)), dtype=torch.uint8)
                out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(out, src, group=group)
                allb = torch.cat(out).numpy()  # keep alive across the copy
                _c.memmove(recv, allb.ctypes.data, nbytes * world)
                return 0
            except Exception:  # reported by the library as DPR_ERR_NCCL
                return 1

        fn = ALLGATHER_FN(_allgather)
        coll = dpr_host_collectives(fn, None)
        alloc = TorchAllocator(cuda_device)
        h = _P()
        _check(load().dpr_create_device_hostcoll(rank, world, cuda_device, _c.byref(coll), _P(stream.cuda_stream),
                                                 _c.byref(alloc.struct), _c.byref(h)))
        dev = cls(h.value, rank, world, alloc, stream)
        dev._keep += [fn, coll]  # the library keeps the function pointer
        return dev

    def release(self):
        if self.h:
            _check(load().dpr_release_device(self.h))
            self.h = None

    # -- world ------------------------------------------------------------------------
    def commit_part(self, part, device_arrays: bool = False, async_copy: bool = False):
        """async_copy=True: DPR_MEMORY_HOST_ASYNC -- the (pinned) host arrays are uploaded on
        a side stream overlapping a render in flight; keep them unchanged until
        commit_world returns."""
        keep: list = []
        desc = part_desc(part, keep, device_arrays, async_copy)
        _check(load().dpr_commit_part(self.h, _c.byref(desc)), self.h)

    def clear_parts(self):
        _check(load().dpr_clear_parts(self.h), self.h)

    def commit_world(self):
        _check(load().dpr_commit_world(self.h), self.h)

    def get_world_bounds(self) -> np.ndarray:
        out = np.zeros(6, np.float32)
        _check(load().dpr_get_world_bounds(self.h, out.ctypes.data), self.h)
        return out

    # -- frame ------------------------------------------------------------------------
    def set_camera(self, cam):
        c = camera_struct(cam)
        _check(load().dpr_set_camera(self.h, _c.byref(c)), self.h)

    def set_frame(self, fr):
        f = frame_struct(fr)
        _check(load().dpr_set_frame(self.h, _c.byref(f)), self.h)

    def render_frame(self):
        _check(load().dpr_render_frame(self.h), self.h)

    def render_frame_composite(self):
        """Compositing contrast device: local renders + deep compositing."""
        _check(load().dpr_render_frame_composite(self.h), self.h)

    def render_frame_replicated(self):
        """Data-replicated mode: whole world on every rank, pixels split."""
        _check(load().dpr_render_frame_replicated(self.h), self.h)

    def frame_ready(self) -> bool:
        return bool(_check(load().dpr_frame_ready(self.h, 1), self.h))

    def map_frame(self):
        """Rank 0: a torch CUDA tensor view (H, W, 4) float32 of the final frame; other
        ranks: None (undefined, not an error)."""
        import torch
        ptr, w, h, und = _P(), _c.c_int(0), _c.c_int(0), _c.c_int(0)
        _check(load().dpr_map_frame(self.h, _c.byref(ptr), _c.byref(w), _c.byref(h), _c.byref(und)), self.h)
        if und.value:
            return None
        return torch.as_tensor(_CudaArray(ptr.value, (h.value, w.value, 4), "<f4"), device="cuda")

    def get_debug(self, spp: int, max_depth: int, npix: int):
        import torch
        ev, oc = _P(), _P()
        _check(load().dpr_get_debug(self.h, _c.byref(ev), _c.byref(oc)), self.h)
        shape = (spp, max_depth, npix)
        return (torch.as_tensor(_CudaArray(ev.value, shape, "<u4"), device="cuda"),
                torch.as_tensor(_CudaArray(oc.value, shape, "<u4"), device="cuda"))

    def get_stats(self) -> dict:
        st = dpr_stats()
        _check(load().dpr_get_stats(self.h, _c.byref(st)), self.h)
        return st.to_dict()

    def get_step_stats(self, max_steps: int = 256) -> dict:
        """dpr_get_step_stats: per-step routing matrices S[k][kind][src][dst], visits
        V[k][kind][rank], step latency and step-barrier time (ms) of the last frame."""
        n = self.nranks
        S = np.zeros((max_steps, 3, n, n), np.int64)
        V = np.zeros((max_steps, 3, n), np.int64)
        ms = np.zeros(max_steps, np.float64)
        sync = np.zeros(max_steps, np.float64)
        ns = _c.c_int(0)
        _check(load().dpr_get_step_stats(self.h, max_steps, S.ctypes.data, V.ctypes.data, ms.ctypes.data,
                                         sync.ctypes.data, _c.byref(ns)), self.h)
        k = min(ns.value, max_steps)
        return {"nsteps": ns.value, "S": S[:k], "V": V[:k], "ms": ms[:k], "sync_ms": sync[:k]}

    def commit_scene_parts(self, parts: Sequence, device_arrays: bool = False):
        for p in parts:
            if p.rank == self.rank:
                self.commit_part(p, device_arrays)


def loopback_group(nranks: int, cuda_device: int = 0, stream=None, torch_alloc: bool = True):
    """dpr_create_loopback_group: N virtual ranks on one GPU (test fixture)."""
    import torch
    torch.cuda.set_device(cuda_device)
    stream = stream or torch.cuda.current_stream(cuda_device)
    alloc = TorchAllocator(cuda_device) if torch_alloc else None
    hs = (_P * nranks)()
    _check(load().dpr_create_loopback_group(nranks, cuda_device, _P(stream.cuda_stream),
                                            _c.byref(alloc.struct) if alloc else None, hs))
    return [Device(hs[r], r, nranks, alloc, stream) for r in range(nranks)]


def render_frame_group(devs: List[Device]):
    arr = (_P * len(devs))(*[d.h for d in devs])
    _check(load().dpr_render_frame_group(arr, len(devs)), devs[0].h)


def render_frame_replicated_group(devs: List[Device]):
    arr = (_P * len(devs))(*[d.h for d in devs])
    _check(load().dpr_render_frame_replicated_group(arr, len(devs)), devs[0].h)


def render_frame_composite_group(devs: List[Device]):
    arr = (_P * len(devs))(*[d.h for d in devs])
    _check(load().dpr_render_frame_composite_group(arr, len(devs)), devs[0].h)
