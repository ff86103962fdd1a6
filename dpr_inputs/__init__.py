"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA product path.

This module holds NONE of the method's arithmetic: no ray generation, tracing, routing or
shading.  It builds scene parts (triangle meshes, spheres, structured-volume bricks), the
camera basis handed to both sides as float32 ("the harness computes the
basis in double ... each component is rounded once to f32"), frame descriptors, and the
application-level partition of a world over ranks (S2.2: "distribute the scene
data in a very simple way").  Every generator is a pure function of its arguments.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdpr_inputs.so")
_lib = None


def build_lib(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-ffp-contract=off",
                               "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build_lib()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.dpri_gyroid_mt.restype = ctypes.c_int64
        _lib.dpri_gyroid_mt.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
        _lib.dpri_volume_field.restype = ctypes.c_int
        _lib.dpri_volume_field.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int]
    return _lib


# ----------------------------------------------------------------------------------------
# Scene description types (mirrors the boundary's dpr_part_desc; include/dpr.h)
# ----------------------------------------------------------------------------------------
TRIS, SPHERES, BRICK = 0, 1, 2


@dataclass
class Part:
    """One rank-local world part (S3.1.2: world content is rank-local)."""
    rank: int
    kind: int
    albedo: Sequence[float] = (0.8, 0.8, 0.8)
    verts: Optional[np.ndarray] = None      # (n,3) float32
    idx: Optional[np.ndarray] = None        # (m,3) int32
    spheres: Optional[np.ndarray] = None    # (n,4) float32: cx cy cz r
    gdims: Sequence[int] = (0, 0, 0)
    origin: Sequence[float] = (0.0, 0.0, 0.0)
    spacing: Sequence[float] = (1.0, 1.0, 1.0)
    cell_lo: Sequence[int] = (0, 0, 0)
    cell_hi: Sequence[int] = (0, 0, 0)
    voxels: Optional[np.ndarray] = None     # float32, x fastest, shape (nz,ny,nx)
    tf: Optional[np.ndarray] = None         # (256,4) float32
    tf_lo: float = 0.0
    tf_hi: float = 1.0
    density_scale: float = 1.0

    def nprims(self) -> int:
        if self.kind == TRIS:
            return int(self.idx.shape[0])
        if self.kind == SPHERES:
            return int(self.spheres.shape[0])
        return 0


@dataclass
class Camera:
    E: np.ndarray
    L: np.ndarray
    U: np.ndarray
    V: np.ndarray
    lens_radius: float = 0.0   # thin-lens depth of field (reading R-DOF); 0 = pinhole
    focus_dist: float = 0.0


@dataclass
class Frame:
    W: int
    H: int
    spp: int = 1
    spp_batch: int = 1
    max_depth: int = 1
    ao_k: int = 0
    ao_radius: float = float("inf")
    light_dir: Sequence[float] = (0.0, 1.0, 0.0)
    E: Sequence[float] = (1.0, 1.0, 1.0)
    A: Sequence[float] = (0.0, 0.0, 0.0)
    B: Sequence[float] = (0.0, 0.0, 0.0)
    dt: float = 0.0
    seed: int = 7
    flags: int = 0   # bit0: fixed jitter 0.5 (test mode)


@dataclass
class Scene:
    name: str
    parts: List[Part]
    nranks: int
    camera: Camera
    frame: Frame
    meta: dict = field(default_factory=dict)


def f32(v) -> np.ndarray:
    return np.asarray(v, dtype=np.float64).astype(np.float32)


def normalize(v) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v)


def camera_basis(pos, look_at, up, fovy_deg: float, W: int, H: int) -> Camera:
    """w=dir/|dir|, u=cross(w,up)/|.|, v=cross(u,w), h=tan(fovy*pi/360);
    U=2h*aspect*u, V=2h*v, L=w-h*aspect*u-h*v; each rounded once to f32; E=pos."""
    pos = np.asarray(pos, np.float64)
    w = normalize(np.asarray(look_at, np.float64) - pos)
    u = np.cross(w, np.asarray(up, np.float64))
    u = u / np.linalg.norm(u)
    v = np.cross(u, w)
    h = math.tan(fovy_deg * math.pi / 360.0)
    aspect = W / H
    return Camera(E=f32(pos), L=f32(w - h * aspect * u - h * v), U=f32(2 * h * aspect * u),
                  V=f32(2 * h * v))


def camera_from_dir(pos, direction, up, fovy_deg, W, H) -> Camera:
    return camera_basis(pos, np.asarray(pos, np.float64) + np.asarray(direction, np.float64),
                        up, fovy_deg, W, H)


# ----------------------------------------------------------------------------------------
# Geometry generators
# ----------------------------------------------------------------------------------------
def gyroid_mesh(G: int, k: float = 4 * math.pi, nthreads: Optional[int] = None):
    """Marching-tetrahedra gyroid on a G^3 point grid over [-1,1]^3 -> indexed mesh
    (verts (nv,3) f32, one per cut grid edge and shared by its triangles; idx (nt,3) i32)."""
    lib = _load()
    nth = nthreads or os.cpu_count() or 1
    nv = ctypes.c_int64(0)
    n = lib.dpri_gyroid_mt(G, k, None, None, 0, 0, nth, ctypes.byref(nv))
    if n < 0:
        raise RuntimeError("gyroid count failed")
    verts = np.empty((nv.value, 3), np.float32)
    idx = np.empty((n, 3), np.int32)
    m = lib.dpri_gyroid_mt(G, k, verts.ctypes.data, idx.ctypes.data, nv.value, n, nth, None)
    if m != n:
        raise RuntimeError("gyroid generation failed")
    return verts, idx


def quad_tris(corners) -> tuple:
    v = f32(corners)
    return v, np.array([[0, 1, 2], [0, 2, 3]], np.int32)


def sphere_clusters(n_clusters: int, per_cluster: int, sigma: float, rmin: float, rmax: float,
                    seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.Philox(seed))
    centres = rng.uniform(-1, 1, size=(n_clusters, 3))
    pts = centres[:, None, :] + sigma * rng.standard_normal((n_clusters, per_cluster, 3))
    r = rng.uniform(rmin, rmax, size=(n_clusters, per_cluster, 1))
    return f32(np.concatenate([pts, r], axis=2).reshape(-1, 4))


def volume_field(G: int, lo=(0, 0, 0), hi=None, nthreads: Optional[int] = None) -> np.ndarray:
    """Procedural field on the G^3 grid over [-1,1]^3; returns the inclusive sub-box
    [lo, hi] as float32 (nz, ny, nx)."""
    lib = _load()
    if hi is None:
        hi = (G - 1, G - 1, G - 1)
    lo = np.asarray(lo, np.int32)
    hi = np.asarray(hi, np.int32)
    shape = tuple(int(x) for x in (hi - lo + 1)[::-1])
    out = np.empty(shape, np.float32)
    lib.dpri_volume_field(G, lo.ctypes.data, hi.ctypes.data, out.ctypes.data,
                          nthreads or os.cpu_count() or 1)
    return out


def default_tf(alpha_max: float = 0.02, s0: float = 0.3) -> np.ndarray:
    """SURVEY 8(d) C3 TF: alpha=0 below s0, rising linearly to alpha_max at s=1; rgb ramp
    blue -> white.  256 entries over [0,1]."""
    s = np.arange(256, dtype=np.float64) / 255.0
    a = np.where(s < s0, 0.0, (s - s0) / (1.0 - s0) * alpha_max)
    rgb = np.stack([s, s, np.ones_like(s)], axis=1) * 0.5 + 0.5 * np.stack([s, s, s], axis=1)
    return f32(np.concatenate([rgb, a[:, None]], axis=1))


# ----------------------------------------------------------------------------------------
# Partitioning (application side)
# ----------------------------------------------------------------------------------------
def bisect_partition(points: np.ndarray, nparts: int) -> np.ndarray:
    """Recursive median bisection of points on the longest axis into nparts groups.
    Returns the group index of each point (stable, deterministic)."""
    n = points.shape[0]
    out = np.zeros(n, np.int32)

    def rec(sel: np.ndarray, first: int, count: int):
        if count == 1 or sel.size == 0:
            out[sel] = first
            return
        p = points[sel]
        ext = p.max(axis=0) - p.min(axis=0)
        ax = int(np.argmax(ext))
        left_parts = count // 2
        k = (sel.size * left_parts) // count
        order = np.lexsort((sel, p[:, ax]))
        rec(sel[order[:k]], first, left_parts)
        rec(sel[order[k:]], first + left_parts, count - left_parts)

    rec(np.arange(n), 0, nparts)
    return out


PARTITIONS = ("spatial", "roundrobin", "binpack")


def partition_groups(cen: np.ndarray, nranks: int, strategy: str = "spatial") -> np.ndarray:
    """Prim -> rank assignment (S2.2: "distribute the scene data in a very simple
    way -- e.g., round-robin, bin-packing until all GPU memory is used").
      spatial    recursive median bisection of centroids (compact rank boxes)
      roundrobin prim i -> rank i mod N (in the mesh's own order)
      binpack    contiguous runs of the input order, equal sizes (fill a rank, then the next)"""
    n = cen.shape[0]
    if strategy == "spatial":
        return bisect_partition(cen, nranks)
    if strategy == "roundrobin":
        return (np.arange(n) % nranks).astype(np.int32)
    if strategy == "binpack":
        return (np.arange(n) * nranks // max(n, 1)).astype(np.int32)
    raise ValueError(strategy)


def split_mesh(verts: np.ndarray, idx: np.ndarray, nranks: int, albedo,
               strategy: str = "spatial") -> List[Part]:
    """Partition of a triangle mesh over ranks (spatial bisection)."""
    cen = tri_centroids(verts, idx)
    grp = partition_groups(cen, nranks, strategy)
    parts = []
    for r in range(nranks):
        v, i = submesh(verts, idx, np.nonzero(grp == r)[0])
        parts.append(Part(rank=r, kind=TRIS, albedo=albedo, verts=v, idx=i))
    return parts


def tri_centroids(verts: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Triangle centroids in float64 (the partitioning key), chunked to bound memory."""
    out = np.empty((idx.shape[0], 3), np.float64)
    for b in range(0, idx.shape[0], 1 << 22):
        out[b:b + (1 << 22)] = verts[idx[b:b + (1 << 22)]].astype(np.float64).mean(axis=1)
    return out


def submesh(verts: np.ndarray, idx: np.ndarray, sel: np.ndarray):
    """Triangles `sel` of an indexed mesh with their vertices compacted (vertex order kept)."""
    t = idx[sel]
    used = np.zeros(verts.shape[0], bool)
    used[t.ravel()] = True
    remap = np.cumsum(used, dtype=np.int64) - 1
    return np.ascontiguousarray(verts[used]), remap[t].astype(np.int32)


def brick_boxes(cells, nparts: int):
    """Recursive bisection of the cell domain [0,cells)^3 into nparts boxes (lo, hi)."""
    boxes = [((0, 0, 0), tuple(cells), nparts)]
    out = []
    while boxes:
        lo, hi, n = boxes.pop(0)
        if n == 1:
            out.append((lo, hi))
            continue
        ext = [hi[c] - lo[c] for c in range(3)]
        ax = int(np.argmax(ext))
        nl = n // 2
        mid = lo[ax] + (ext[ax] * nl) // n
        hl = list(hi); hl[ax] = mid
        lr = list(lo); lr[ax] = mid
        boxes.append((lo, tuple(hl), nl))
        boxes.append((tuple(lr), hi, n - nl))
    return out


def volume_bricks(G: int, nranks: int, tf: np.ndarray, density_scale: float = 1.0,
                  field_fn=None) -> List[Part]:
    """Split the G^3 grid ((G-1)^3 cells) into nranks bricks; each brick stores voxels
    [cell_lo, cell_hi] inclusive (one ghost layer).  Origin -1, spacing 2/(G-1)."""
    h = np.float32(2.0 / (G - 1))
    parts = []
    boxes = brick_boxes((G - 1, G - 1, G - 1), nranks)
    for r, (lo, hi) in enumerate(boxes):
        vox = (field_fn or volume_field)(G, lo, hi)
        parts.append(Part(rank=r, kind=BRICK, albedo=(1, 1, 1), gdims=(G, G, G),
                          origin=(-1.0, -1.0, -1.0), spacing=(float(h),) * 3, cell_lo=lo,
                          cell_hi=hi, voxels=np.ascontiguousarray(vox), tf=tf, tf_lo=0.0,
                          tf_hi=1.0, density_scale=density_scale))
    return parts


def reassign(parts: List[Part], nranks: int) -> List[Part]:
    return [replace(p, rank=p.rank % nranks) for p in parts]


def union_parts(parts: List[Part]) -> List[Part]:
    """The merged world on one rank, in rank order (global ids of the
    union are the concatenation in rank order)."""
    out = []
    for r in sorted({p.rank for p in parts}):
        out += [replace(p, rank=0) for p in parts if p.rank == r]
    return out


# ----------------------------------------------------------------------------------------
# Configs (BASELINE.json configs; concretised in SURVEY 8(d))
# ----------------------------------------------------------------------------------------
C1_SPHERES = [((-1.5, 0.5, 0.0), 0.5, (0.9, 0.2, 0.2)),
              ((-0.6, 0.8, 1.2), 0.8, (0.2, 0.9, 0.2)),
              ((0.9, 0.4, -0.8), 0.4, (0.2, 0.2, 0.9)),
              ((1.8, 1.0, 0.7), 1.0, (0.9, 0.9, 0.2))]


def config1(W: int = 64, H: int = 64) -> Scene:
    """configs[0]: two-rank world of 4 spheres + ground plane split by x-half, 64x64, 1 spp,
    AO 4 rays, depth 2."""
    parts = []
    for r, (x0, x1) in enumerate([(-4.0, 0.0), (0.0, 4.0)]):
        v, i = quad_tris([(x0, 0, -4), (x1, 0, -4), (x1, 0, 4), (x0, 0, 4)])
        parts.append(Part(rank=r, kind=TRIS, albedo=(0.8, 0.8, 0.8), verts=v, idx=i))
    for j, (c, rad, rho) in enumerate(C1_SPHERES):
        r = 0 if j < 2 else 1
        parts.append(Part(rank=r, kind=SPHERES, albedo=rho,
                          spheres=f32([[c[0], c[1], c[2], rad]])))
    # commit order within a rank: ground half, then its spheres
    parts = [parts[0], parts[2], parts[3], parts[1], parts[4], parts[5]]
    cam = camera_basis((0, 2.5, -7), (0, 0.6, 0), (0, 1, 0), 40.0, W, H)
    fr = Frame(W=W, H=H, spp=1, spp_batch=1, max_depth=2, ao_k=4, ao_radius=float("inf"),
               light_dir=f32(normalize((1, 0.8, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3),
               B=(0.05, 0.05, 0.1), seed=7)
    return Scene("C1", parts, 2, cam, fr)


C2_G = 301


def config2(nranks: int = 1, G: int = C2_G, W: int = 1024, H: int = 1024, spp: int = 16,
            spp_batch: int = 16, partition: str = "spatial") -> Scene:
    """configs[1]: synthetic ~10M-triangle gyroid spatially partitioned over N ranks,
    1024x1024, 16 spp, shadows + AO (K=4, aoRadius 0.25, depth 1)."""
    verts, idx = gyroid_mesh(G)
    parts = split_mesh(verts, idx, nranks, (0.75, 0.75, 0.75), partition)
    cam = camera_basis((2.2, 1.6, 2.8), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    fr = Frame(W=W, H=H, spp=spp, spp_batch=spp_batch, max_depth=1, ao_k=4, ao_radius=0.25,
               light_dir=f32(normalize((1, 1.5, 0.5))), E=(1, 1, 1), A=(0.4, 0.4, 0.4),
               B=(0.05, 0.05, 0.05), seed=7)
    return Scene("C2", parts, nranks, cam, fr, meta={"G": G, "ntris": int(idx.shape[0])})


def config3(nranks: int = 1, G: int = 1024, W: int = 1920, H: int = 1080) -> Scene:
    """configs[2]: structured G^3 float32 volume split into per-rank bricks, DVR with volume
    shadows (1 spp, depth 1), 1920x1080."""
    tf = default_tf()
    parts = volume_bricks(G, nranks, tf)
    cam = camera_basis((0, 0.5, 3.2), (0, 0, 0), (0, 1, 0), 40.0, W, H)
    h = float(np.float32(2.0 / (G - 1)))
    fr = Frame(W=W, H=H, spp=1, spp_batch=1, max_depth=1, ao_k=0, ao_radius=0.0,
               light_dir=f32(normalize((1, 2, 1))), E=(1, 1, 1), A=(0, 0, 0), B=(0, 0, 0),
               dt=h, seed=7)
    return Scene("C3", parts, nranks, cam, fr, meta={"G": G})


def cluster_palette(n: int, seed: int = 11) -> np.ndarray:
    rng = np.random.Generator(np.random.Philox(seed))
    return f32(0.25 + 0.7 * rng.uniform(size=(n, 3)))


def partition_parts_mixed(sph: np.ndarray, sph_cluster: np.ndarray, palette: np.ndarray,
                          verts: np.ndarray, idx: np.ndarray, mesh_albedo, nranks: int) -> List[Part]:
    """Bisection of the centroids of ALL prims (spheres + triangles) into nranks groups;
    within a rank: the mesh part, then one sphere part per cluster (commit order)."""
    cen = np.concatenate([sph[:, :3].astype(np.float64), tri_centroids(verts, idx)])
    grp = bisect_partition(cen, nranks) if nranks > 1 else np.zeros(cen.shape[0], np.int32)
    gs, gt = grp[:sph.shape[0]], grp[sph.shape[0]:]
    parts = []
    for r in range(nranks):
        tsel = np.nonzero(gt == r)[0]
        if tsel.size:
            v, i = submesh(verts, idx, tsel)
            parts.append(Part(rank=r, kind=TRIS, albedo=mesh_albedo, verts=v, idx=i))
        sel = np.nonzero(gs == r)[0]
        cl = sph_cluster[sel]
        order = np.argsort(cl, kind="stable")
        sel, cl = sel[order], cl[order]
        bounds = np.flatnonzero(np.diff(cl)) + 1
        for chunk in np.split(np.arange(sel.size), bounds):
            if chunk.size == 0:
                continue
            c = int(cl[chunk[0]])
            parts.append(Part(rank=r, kind=SPHERES, albedo=palette[c],
                              spheres=np.ascontiguousarray(sph[sel[chunk]])))
    return parts


def config4(nranks: int = 8, n_clusters: int = 1000, per_cluster: int = 50_000, G: int = 211,
            W: int = 1920, H: int = 1080, spp: int = 1) -> Scene:
    """configs[3]: mixed scene -- 50M spheres (1000 Gaussian clusters, sigma 0.05, r in
    [0.002, 0.004]) + a gyroid iso-surface (G=211, ~5M triangles) over N ranks by centroid
    bisection; path tracing depth 4, one AO ray (r=0.1), shadow + bounce per vertex."""
    sph = sphere_clusters(n_clusters, per_cluster, 0.05, 0.002, 0.004, seed=5)
    cl = np.repeat(np.arange(n_clusters, dtype=np.int32), per_cluster)
    verts, idx = gyroid_mesh(G)
    parts = partition_parts_mixed(sph, cl, cluster_palette(n_clusters), verts, idx, (0.75, 0.75, 0.75),
                                  nranks)
    cam = camera_basis((2.2, 1.6, 2.8), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    fr = Frame(W=W, H=H, spp=spp, spp_batch=spp, max_depth=4, ao_k=1, ao_radius=0.1,
               light_dir=f32(normalize((1, 1.5, 0.5))), E=(1, 1, 1), A=(0.4, 0.4, 0.4),
               B=(0.05, 0.05, 0.05), seed=7)
    return Scene("C4", parts, nranks, cam, fr,
                 meta={"spheres": int(sph.shape[0]), "ntris": int(idx.shape[0])})


def config5(nranks: int = 8, G_mesh: int = 950, G_vol: int = 1024, W: int = 3840, H: int = 2160,
            spp: int = 64, spp_batch: int = 4, alpha_max: float = 0.02) -> Scene:
    """configs[4]: 4K, 64 spp, ~100M-triangle gyroid + the 1024^3 volume bricks over N ranks
    (depth 2, K=1, aoRadius 0.25, batches of 4 spp)."""
    verts, idx = gyroid_mesh(G_mesh)
    parts = split_mesh(verts, idx, nranks, (0.75, 0.75, 0.75))
    parts += volume_bricks(G_vol, nranks, default_tf(alpha_max=alpha_max))
    cam = camera_basis((2.2, 1.6, 2.8), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    h = float(np.float32(2.0 / (G_vol - 1)))
    fr = Frame(W=W, H=H, spp=spp, spp_batch=spp_batch, max_depth=2, ao_k=1, ao_radius=0.25,
               light_dir=f32(normalize((1, 1.5, 0.5))), E=(1, 1, 1), A=(0.4, 0.4, 0.4),
               B=(0.05, 0.05, 0.05), dt=h, seed=7)
    return Scene("C5", parts, nranks, cam, fr, meta={"ntris": int(idx.shape[0]), "G_vol": G_vol})


def box_tris(lo, hi) -> np.ndarray:
    """12 triangles of an axis-aligned box, (12, 3, 3) float32."""
    x0, y0, z0 = lo
    x1, y1, z1 = hi
    c = np.array([[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0],
                  [x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]], np.float64)
    f = [(0, 1, 2), (0, 2, 3), (4, 6, 5), (4, 7, 6), (0, 4, 5), (0, 5, 1),
         (3, 2, 6), (3, 6, 7), (0, 3, 7), (0, 7, 4), (1, 5, 6), (1, 6, 2)]
    return f32(c[np.array(f)])


def boxes_scene(nranks: int = 4, n: int = 4, W: int = 256, H: int = 256, spp: int = 4,
                seed: int = 3) -> Scene:
    """PAPER Fig. composite-tests-diffuse (E5): 4^3 boxes pseudo-randomly
    interleaved across 4 ranks, on a ground plane (rank 0), lit from the side so that boxes
    of one rank shadow boxes and ground of another -- the global shadows a compositing device
    cannot produce."""
    rng = np.random.Generator(np.random.Philox(seed))
    owner = rng.integers(0, nranks, size=n ** 3)
    palette = cluster_palette(nranks, seed=seed + 1)
    tris = [[] for _ in range(nranks)]
    k = 0
    step = 1.6 / n
    for ix in range(n):
        for iy in range(n):
            for iz in range(n):
                lo = (-0.8 + ix * step + 0.05, -0.8 + iy * step + 0.05, -0.8 + iz * step + 0.05)
                hi = (lo[0] + step * 0.62, lo[1] + step * 0.62, lo[2] + step * 0.62)
                tris[owner[k]].append(box_tris(lo, hi))
                k += 1
    parts = []
    for r in range(nranks):
        if r == 0:
            gv, gi = quad_tris([(-3, -0.85, -3), (3, -0.85, -3), (3, -0.85, 3), (-3, -0.85, 3)])
            parts.append(Part(rank=0, kind=TRIS, albedo=(0.8, 0.8, 0.8), verts=gv, idx=gi))
        if tris[r]:
            t = np.concatenate(tris[r]).reshape(-1, 3)
            parts.append(Part(rank=r, kind=TRIS, albedo=palette[r], verts=t,
                              idx=np.arange(t.shape[0], dtype=np.int32).reshape(-1, 3)))
    cam = camera_basis((2.6, 1.9, 3.3), (0, -0.2, 0), (0, 1, 0), 40.0, W, H)
    fr = Frame(W=W, H=H, spp=spp, spp_batch=spp, max_depth=2, ao_k=2, ao_radius=0.5,
               light_dir=f32(normalize((-1.0, 1.4, 0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3),
               B=(0.1, 0.1, 0.15), seed=7)
    return Scene("E5", parts, nranks, cam, fr)


def routing_hand_case(which: str) -> Scene:
    """SURVEY 8(c).4 hand cases H1-H3 (1x1 image, jitter 0.5, d = (0,0,1) exactly), plus H4:
    the eye (0.2,0.2,-1) lies inside BOTH padded rank boxes (each rank also owns a tiny
    triangle at z=-2 off the ray's path), so the primary's entry distance is t0=0 for both
    ranks -- the equal-t0 tie of the visit key (t0_r, r); and H5: rank 0's square sits at
    z = 2.0001f, so its padded box is entered at exactly t0 = 3 = bestT of rank 1's hit (the
    `t0_r <= bestT` bound of P8 taken with equality)."""
    cam = Camera(E=f32((0.2, 0.2, -1)), L=f32((-0.05, -0.05, 1)), U=f32((0.1, 0, 0)),
                 V=f32((0, 0.1, 0)))
    z0 = 2.0001 if which == "H5" else 3.0
    r0 = Part(rank=0, kind=TRIS, albedo=(0.5, 0.6, 0.7),
              verts=f32([(-1, -1, z0), (1, -1, z0), (1, 1, z0), (-1, 1, z0)]),
              idx=np.array([[0, 1, 2], [0, 2, 3]], np.int32))
    if which in ("H1", "H3", "H4"):
        r1v = f32([(-.5, -.5, 2), (.5, -.5, 2), (-.5, .5, 2)])
    else:  # H2, H5: rank 1's triangle covers (0.2, 0.2)
        r1v = f32([(-.5, -.5, 2), (1, -.5, 2), (-.5, 1, 2)])
    r1 = Part(rank=1, kind=TRIS, albedo=(0.9, 0.3, 0.1), verts=r1v,
              idx=np.array([[0, 1, 2]], np.int32))
    parts = [r0, r1]
    if which == "H4":
        parts += [Part(rank=0, kind=TRIS, albedo=(0.1, 0.1, 0.1),
                       verts=f32([(-1, -1, -2), (-.9, -1, -2), (-1, -.9, -2)]),
                       idx=np.array([[0, 1, 2]], np.int32)),
                  Part(rank=1, kind=TRIS, albedo=(0.1, 0.1, 0.1),
                       verts=f32([(.9, .9, -2), (1, .9, -2), (1, 1, -2)]),
                       idx=np.array([[0, 1, 2]], np.int32))]
    l = (0, 0, 1) if which == "H3" else (0, 0, -1)
    fr = Frame(W=1, H=1, spp=1, spp_batch=1, max_depth=1, ao_k=0, light_dir=f32(l),
               E=(1, 1, 1), A=(0, 0, 0), B=(0, 0, 0), seed=7, flags=1)
    return Scene(which, parts, 2, cam, fr)
