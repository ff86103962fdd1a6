"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package.  The product path (paper_2407_00179_b200/) never imports
it, and the two share no code; both consume dpr_inputs (seeded synthetic inputs only).

This module is argument marshalling for oracle/dpr_oracle.c (see its header for what is
computed and which PAPER.md passages each function follows).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

import dpr_inputs as di

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dpr_oracle.c")
LIB_PATH = os.path.join(_HERE, "liboracle.so")
# tools/oracle_mutations.py points this at a mutated build (checks that each pin can fail)
_LIB_OVERRIDE = os.environ.get("DPR_ORACLE_LIB")
_lib = None

CFLAGS = ["-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
          "-fPIC", "-shared", "-pthread", "-fvisibility=hidden"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB_PATH, _SRC, "-lm"])
    return LIB_PATH


class or_part(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("kind", ctypes.c_int32),
                ("albedo", ctypes.c_float * 3),
                ("n_verts", ctypes.c_int64), ("verts", ctypes.c_void_p),
                ("n_tris", ctypes.c_int64), ("idx", ctypes.c_void_p),
                ("n_spheres", ctypes.c_int64), ("spheres", ctypes.c_void_p),
                ("gdims", ctypes.c_int32 * 3), ("origin", ctypes.c_float * 3),
                ("spacing", ctypes.c_float * 3), ("cell_lo", ctypes.c_int32 * 3),
                ("cell_hi", ctypes.c_int32 * 3), ("voxels", ctypes.c_void_p),
                ("tf", ctypes.c_void_p), ("tf_lo", ctypes.c_float), ("tf_hi", ctypes.c_float),
                ("density_scale", ctypes.c_float)]


class or_camera(ctypes.Structure):
    _fields_ = [("E", ctypes.c_float * 3), ("L", ctypes.c_float * 3),
                ("U", ctypes.c_float * 3), ("V", ctypes.c_float * 3),
                ("lens_radius", ctypes.c_float), ("focus_dist", ctypes.c_float)]


class or_frame(ctypes.Structure):
    _fields_ = [("W", ctypes.c_int32), ("H", ctypes.c_int32), ("spp", ctypes.c_int32),
                ("spp_batch", ctypes.c_int32), ("max_depth", ctypes.c_int32),
                ("ao_k", ctypes.c_int32), ("ao_radius", ctypes.c_float),
                ("light_dir", ctypes.c_float * 3), ("E", ctypes.c_float * 3),
                ("A", ctypes.c_float * 3), ("B", ctypes.c_float * 3), ("dt", ctypes.c_float),
                ("seed", ctypes.c_uint64), ("flags", ctypes.c_int32)]


_P = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        if _LIB_OVERRIDE:
            L = ctypes.CDLL(_LIB_OVERRIDE)
        else:
            build()
            L = ctypes.CDLL(LIB_PATH)
        L.or_scene_build.restype = _P
        L.or_scene_build.argtypes = [_P, ctypes.c_int, ctypes.c_int]
        L.or_scene_free.argtypes = [_P]
        L.or_scene_nprims.restype = ctypes.c_int64
        L.or_scene_nprims.argtypes = [_P]
        L.or_scene_rank_box.argtypes = [_P, ctypes.c_int, _P, _P]
        for fn in (L.or_render_union,):
            fn.restype = ctypes.c_int
            fn.argtypes = [_P, _P, _P, _P, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_int]
        L.or_render_dp.restype = ctypes.c_int
        L.or_render_dp.argtypes = [_P, _P, _P, _P, ctypes.c_int64, _P, _P, _P, _P, _P, _P, _P,
                                   ctypes.c_int]
        L.or_render_dp_steps.restype = ctypes.c_int
        L.or_render_dp_steps.argtypes = [_P, _P, _P, _P, ctypes.c_int64, _P, _P, _P, _P, _P, _P, _P,
                                         _P, _P, ctypes.c_int, ctypes.c_int]
        L.or_set_brute.argtypes = [ctypes.c_int]
        L.or_render_union_depth.restype = ctypes.c_int
        L.or_render_union_depth.argtypes = [_P, _P, _P, _P, ctypes.c_int64, _P, _P, ctypes.c_int]
        L.or_philox.argtypes = [_P, _P, _P]
        L.or_u01.restype = ctypes.c_float
        L.or_u01.argtypes = [ctypes.c_uint32]
        L.or_tri_hit.restype = ctypes.c_int
        L.or_tri_hit.argtypes = [_P, _P, ctypes.c_float, _P, _P, _P, _P, _P]
        L.or_sphere_hit.restype = ctypes.c_int
        L.or_sphere_hit.argtypes = [_P, _P, ctypes.c_float, _P, ctypes.c_float, _P, _P]
        L.or_slab.restype = ctypes.c_int
        L.or_slab.argtypes = [_P, _P, _P, _P, ctypes.c_float, _P, _P]
        L.or_camera_ray.argtypes = [_P, _P, ctypes.c_uint32, ctypes.c_uint32, _P, _P]
        L.or_cosine_dir.argtypes = [_P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _P]
        L.or_iso_dir.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                 ctypes.c_uint32, _P]
        L.or_ao_dir.argtypes = [_P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                ctypes.c_uint32, ctypes.c_int, _P]
        L.or_bounce_dir.argtypes = [_P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.c_uint32, _P]
        L.or_vol_u.restype = ctypes.c_float
        L.or_vol_u.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                               ctypes.c_int, ctypes.c_int, ctypes.c_int64]
        L.or_pln.restype = ctypes.c_float
        L.or_pln.argtypes = [ctypes.c_float]
        L.or_tf_eval.argtypes = [_P, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                 ctypes.c_float, _P]
        L.or_brick_sample.restype = ctypes.c_int
        L.or_brick_sample.argtypes = [_P, _P, _P]
        for fn in (L.or_brute_closest, L.or_bvh_closest):
            fn.argtypes = [_P, _P, _P, ctypes.c_float, _P, _P]
        for fn in (L.or_brute_any, L.or_bvh_any):
            fn.restype = ctypes.c_int
            fn.argtypes = [_P, _P, _P, ctypes.c_float]
        _lib = L
    return _lib


def _fa(v, n=3):
    return (ctypes.c_float * n)(*[float(x) for x in v])


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def make_part(p: di.Part, keep: list) -> or_part:
    s = or_part()
    s.rank, s.kind = p.rank, p.kind
    s.albedo = _fa(p.albedo)
    if p.kind == di.TRIS:
        v = np.ascontiguousarray(p.verts, np.float32)
        i = np.ascontiguousarray(p.idx, np.int32)
        keep += [v, i]
        s.n_verts, s.verts, s.n_tris, s.idx = v.shape[0], _ptr(v), i.shape[0], _ptr(i)
    elif p.kind == di.SPHERES:
        sp = np.ascontiguousarray(p.spheres, np.float32)
        keep.append(sp)
        s.n_spheres, s.spheres = sp.shape[0], _ptr(sp)
    else:
        vx = np.ascontiguousarray(p.voxels, np.float32)
        tf = np.ascontiguousarray(p.tf, np.float32)
        keep += [vx, tf]
        s.gdims = (ctypes.c_int32 * 3)(*p.gdims)
        s.origin, s.spacing = _fa(p.origin), _fa(p.spacing)
        s.cell_lo = (ctypes.c_int32 * 3)(*p.cell_lo)
        s.cell_hi = (ctypes.c_int32 * 3)(*p.cell_hi)
        s.voxels, s.tf = _ptr(vx), _ptr(tf)
        s.tf_lo, s.tf_hi, s.density_scale = p.tf_lo, p.tf_hi, p.density_scale
    return s


def make_camera(c: di.Camera) -> or_camera:
    o = or_camera()
    o.E, o.L, o.U, o.V = _fa(c.E), _fa(c.L), _fa(c.U), _fa(c.V)
    o.lens_radius, o.focus_dist = float(c.lens_radius), float(c.focus_dist)
    return o


def make_frame(f: di.Frame) -> or_frame:
    o = or_frame()
    o.W, o.H, o.spp, o.spp_batch, o.max_depth, o.ao_k = f.W, f.H, f.spp, f.spp_batch, f.max_depth, f.ao_k
    o.ao_radius = f.ao_radius
    o.light_dir, o.E, o.A, o.B = _fa(f.light_dir), _fa(f.E), _fa(f.A), _fa(f.B)
    o.dt = f.dt
    o.seed = f.seed
    o.flags = f.flags
    return o


class OracleScene:
    """Union + per-rank BVHs over a list of parts (global ids per SURVEY 8(c) P12)."""

    def __init__(self, parts: List[di.Part], nranks: int):
        self._keep: list = []
        arr = (or_part * max(1, len(parts)))(*[make_part(p, self._keep) for p in parts])
        self._arr = arr
        self.nranks = nranks
        self.h = lib().or_scene_build(ctypes.addressof(arr), len(parts), nranks)
        if not self.h:
            raise ValueError("or_scene_build failed")

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().or_scene_free(self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    @property
    def nprims(self) -> int:
        return int(lib().or_scene_nprims(self.h))

    def rank_box(self, r: int):
        out = np.zeros(6, np.float32)
        ne = ctypes.c_int(0)
        lib().or_scene_rank_box(self.h, r, out.ctypes.data, ctypes.byref(ne))
        return out, bool(ne.value)

    def closest(self, o, d, tmax=np.inf, brute=False):
        t = ctypes.c_float(0)
        i = ctypes.c_uint32(0)
        fn = lib().or_brute_closest if brute else lib().or_bvh_closest
        fn(self.h, _fa(o), _fa(d), tmax, ctypes.byref(t), ctypes.byref(i))
        return t.value, i.value

    def any_hit(self, o, d, tmax, brute=False):
        fn = lib().or_brute_any if brute else lib().or_bvh_any
        return bool(fn(self.h, _fa(o), _fa(d), tmax))


@dataclass
class RenderResult:
    rgba: np.ndarray                  # (npix,4) float64: sum/spp; alpha = coverage
    events: Optional[np.ndarray]      # (spp, max_depth, npix) uint32
    occl: Optional[np.ndarray]
    gen: np.ndarray                   # rays generated per kind (path, shadow, ao)
    S: Optional[np.ndarray] = None    # (3,N,N) routing matrix
    V: Optional[np.ndarray] = None    # (3,N) visits
    steps: Optional[np.ndarray] = None  # per spp batch
    S_step: Optional[np.ndarray] = None  # (total steps, 3, N, N): per-step routing (P8b), batches in order
    V_step: Optional[np.ndarray] = None  # (total steps, 3, N)


MAX_STEPS_PER_BATCH = 128


def render(scene: OracleScene, cam: di.Camera, fr: di.Frame, pixels=None, dp: bool = False,
           dumps: bool = True, nthreads: int = 0, step_matrices: bool = False) -> RenderResult:
    """Render the listed pixel indices (all samples each); pixels=None -> whole frame.
    step_matrices (dp only): also the per-step routing matrices / visits of P8b."""
    if pixels is None:
        pixels = np.arange(fr.W * fr.H, dtype=np.int64)
    pixels = np.ascontiguousarray(pixels, np.int64)
    n = pixels.size
    c, f = make_camera(cam), make_frame(fr)
    rgba = np.zeros((n, 4), np.float64)
    ev = np.zeros((fr.spp, fr.max_depth, n), np.uint32) if dumps else None
    oc = np.zeros((fr.spp, fr.max_depth, n), np.uint32) if dumps else None
    gen = np.zeros(3, np.int64)
    N = scene.nranks
    if dp:
        S = np.zeros((3, N, N), np.int64)
        V = np.zeros((3, N), np.int64)
        nb = (fr.spp + fr.spp_batch - 1) // fr.spp_batch
        steps = np.zeros(nb, np.int64)
        if step_matrices:
            M = MAX_STEPS_PER_BATCH
            Ss = np.zeros((nb, M, 3, N, N), np.int64)
            Vs = np.zeros((nb, M, 3, N), np.int64)
            rc = lib().or_render_dp_steps(scene.h, ctypes.byref(c), ctypes.byref(f), pixels.ctypes.data, n,
                                          rgba.ctypes.data, _ptr(ev), _ptr(oc), S.ctypes.data, V.ctypes.data,
                                          gen.ctypes.data, steps.ctypes.data, Ss.ctypes.data, Vs.ctypes.data,
                                          M, nthreads)
            if rc != 0:
                raise ValueError("or_render_dp_steps failed")
            if steps.max(initial=0) > M:
                raise ValueError("more steps per batch than MAX_STEPS_PER_BATCH")
            S_step = np.concatenate([Ss[b, :steps[b]] for b in range(nb)])
            V_step = np.concatenate([Vs[b, :steps[b]] for b in range(nb)])
            return RenderResult(rgba, ev, oc, gen, S, V, steps, S_step, V_step)
        rc = lib().or_render_dp(scene.h, ctypes.byref(c), ctypes.byref(f), pixels.ctypes.data, n,
                                rgba.ctypes.data, _ptr(ev), _ptr(oc), S.ctypes.data,
                                V.ctypes.data, gen.ctypes.data, steps.ctypes.data, nthreads)
        if rc != 0:
            raise ValueError("or_render_dp failed")
        return RenderResult(rgba, ev, oc, gen, S, V, steps)
    rc = lib().or_render_union(scene.h, ctypes.byref(c), ctypes.byref(f), pixels.ctypes.data, n,
                               rgba.ctypes.data, _ptr(ev), _ptr(oc), gen.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError("or_render_union failed")
    return RenderResult(rgba, ev, oc, gen)


FLAG_NO_BACKGROUND = 4


def render_local_fragments(parts: List[di.Part], rank: int, cam: di.Camera, fr: di.Frame,
                           nthreads: int = 0):
    """The colour + depth buffers of one rank's LOCAL render (only its own parts, local
    shading, no background) -- what a pass-through device hands to the compositing device
    (S5.1.2).  rgba premultiplied by coverage (= sum/spp), depth = min primary t."""
    local = [di.Part(**{**p.__dict__, "rank": 0}) for p in parts if p.rank == rank]
    sc = OracleScene(local, 1)
    f = di.Frame(**{**fr.__dict__, "flags": fr.flags | FLAG_NO_BACKGROUND})
    n = f.W * f.H
    pix = np.arange(n, dtype=np.int64)
    rgba = np.zeros((n, 4), np.float64)
    depth = np.zeros(n, np.float32)
    c, ff = make_camera(cam), make_frame(f)
    rc = lib().or_render_union_depth(sc.h, ctypes.byref(c), ctypes.byref(ff), pix.ctypes.data, n,
                                     rgba.ctypes.data, depth.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError("or_render_union_depth failed")
    return rgba, depth


def deep_composite(rgba: np.ndarray, depth: np.ndarray, background) -> np.ndarray:
    """deepComp (S5.1.1): per pixel, sort the N ranks' RGBA-z fragments by depth
    (ties: lower rank first) and composite front to back with the over operator on
    premultiplied colour; the background fills the remaining transparency.
    rgba: (N, P, 4) premultiplied, depth: (N, P).  Returns (P, 4)."""
    N, P = depth.shape
    order = np.lexsort((np.broadcast_to(np.arange(N)[:, None], (N, P)), depth), axis=0)
    C = np.zeros((P, 3))
    A = np.zeros(P)
    cols = np.arange(P)
    for k in range(N):
        f = rgba[order[k], cols]
        C += (1.0 - A)[:, None] * f[:, :3]
        A += (1.0 - A) * f[:, 3]
    C += (1.0 - A)[:, None] * np.asarray(background, np.float64)[None, :]
    return np.concatenate([C, A[:, None]], axis=1)


def set_brute(on: bool):
    """Trace by brute force over all prims instead of the oracle BVH (tests / debugging)."""
    lib().or_set_brute(1 if on else 0)


# ---- single-operation wrappers (used by the pin tests) ----------------------------------
def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().or_philox(c, k, o)
    return list(o)


def u01(x: int) -> float:
    return lib().or_u01(x)


def tri_hit(o, d, v0, v1, v2, tmax=np.inf):
    t = ctypes.c_float(0)
    n = (ctypes.c_float * 3)()
    ok = lib().or_tri_hit(_fa(o), _fa(d), tmax, _fa(v0), _fa(v1), _fa(v2), ctypes.byref(t), n)
    return (t.value, list(n)) if ok else None


def sphere_hit(o, d, c, r, tmax=np.inf):
    t = ctypes.c_float(0)
    n = (ctypes.c_float * 3)()
    ok = lib().or_sphere_hit(_fa(o), _fa(d), tmax, _fa(c), r, ctypes.byref(t), n)
    return (t.value, list(n)) if ok else None


def slab(lo, hi, o, d, tmax=np.inf):
    t0, t1 = ctypes.c_float(0), ctypes.c_float(0)
    ok = lib().or_slab(_fa(lo), _fa(hi), _fa(o), _fa(d), tmax, ctypes.byref(t0), ctypes.byref(t1))
    return bool(ok), t0.value, t1.value


def camera_ray(cam: di.Camera, fr: di.Frame, p: int, s: int = 0):
    o, d = (ctypes.c_float * 3)(), (ctypes.c_float * 3)()
    c, f = make_camera(cam), make_frame(fr)
    lib().or_camera_ray(ctypes.byref(c), ctypes.byref(f), p, s, o, d)
    return np.array(o, np.float32), np.array(d, np.float32)


def cosine_dir(n, seed, p, s, depth, purpose, subhi):
    out = (ctypes.c_float * 3)()
    lib().or_cosine_dir(_fa(n), seed, p, s, depth, purpose, subhi, out)
    return np.array(out, np.float32)


def iso_dir(seed, p, s, depth):
    out = (ctypes.c_float * 3)()
    lib().or_iso_dir(seed, p, s, depth, out)
    return np.array(out, np.float32)


def ao_dir(n, seed, p, s, depth, k):
    """AO ray k's direction as the renderer draws it (P1 purpose 2, sub = (k<<4)|attempt)."""
    out = (ctypes.c_float * 3)()
    lib().or_ao_dir(_fa(n), seed, p, s, depth, k, out)
    return np.array(out, np.float32)


def bounce_dir(n, seed, p, s, depth):
    """The bounce direction as the renderer draws it (P1 purpose 3, sub = attempt)."""
    out = (ctypes.c_float * 3)()
    lib().or_bounce_dir(_fa(n), seed, p, s, depth, out)
    return np.array(out, np.float32)


def vol_u(seed, p, s, depth, kind, k, i):
    """u_i of volume sample i of a ray of kind 0 path / 1 shadow / 2 AO k (P1 4/5/6)."""
    return float(lib().or_vol_u(seed, p, s, depth, kind, k, i))


def pln(x: float) -> float:
    """Reading R-LOG: the pinned binary32 natural log used by delta tracking."""
    return float(lib().or_pln(float(x)))


def tf_eval(tf: np.ndarray, lo, hi, dscale, s):
    tf = np.ascontiguousarray(tf, np.float32)
    out = (ctypes.c_float * 4)()
    lib().or_tf_eval(tf.ctypes.data, lo, hi, dscale, s, out)
    return np.array(out, np.float32)


def brick_sample(part: di.Part, p):
    keep: list = []
    s = make_part(part, keep)
    v = ctypes.c_float(0)
    ok = lib().or_brick_sample(ctypes.byref(s), _fa(p), ctypes.byref(v))
    return v.value if ok else None
