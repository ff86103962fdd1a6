"""Oracle pins, part 1: single operations checked against values fixed OUTSIDE the oracle
(published KATs, SPEC worked examples, closed forms, brute force, distributional facts).

Each test names the passage it pins.  P:<n> = PAPER.md line, S:<n> = SPEC.md line,
SURVEY 8(c) Pn = the pinned reading of the paper-silent arithmetic (DESIGN.md readings).
"""
import math
import os

import numpy as np
import pytest

import dpr_inputs as di
import oracle as orc


def test_philox_known_answers(golden_dir):
    """P1: Random123 philox4x32-10 KATs (tests/golden/philox_kat.txt)."""
    n = 0
    for line in open(os.path.join(golden_dir, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        assert orc.philox(w[0:4], w[4:6]) == w[6:10]
        n += 1
    assert n == 3


def test_u01_range_exact():
    """P1: u = (x>>8)*2^-24 lies in [0, 1-2^-24] exactly."""
    assert orc.u01(0) == 0.0
    assert orc.u01(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    assert orc.u01(0x80000000) == 0.5
    assert orc.u01(0x000000FF) == 0.0


def test_sphere_worked_example():
    """ray (0,0,-3)->(0,0,1) vs unit sphere -> t=2, n=(0,0,-1)."""
    t, n = orc.sphere_hit((0, 0, -3), (0, 0, 1), (0, 0, 0), 1.0)
    assert t == 2.0 and n == [0.0, 0.0, -1.0]
    # origin inside: the far root is taken (P4 "if !(t>0) then t=-b+sq")
    t, n = orc.sphere_hit((0, 0, 0), (0, 0, 1), (0, 0, 0), 1.0)
    assert t == 1.0 and n == [0.0, 0.0, -1.0]  # normal oriented against the ray
    assert orc.sphere_hit((0, 2, -3), (0, 0, 1), (0, 0, 0), 1.0) is None
    assert orc.sphere_hit((0, 0, -3), (0, 0, 1), (0, 0, 0), 1.0, tmax=2.0) is None  # t<tmax strict


def test_triangle_worked_example():
    """(0.25,0.25,-1)+(0,0,1) vs (0,0,0),(1,0,0),(0,1,0) -> t=1 (double-sided)."""
    t, n = orc.tri_hit((0.25, 0.25, -1), (0, 0, 1), (0, 0, 0), (1, 0, 0), (0, 1, 0))
    assert t == 1.0 and abs(n[2] + 1.0) == 0.0
    t2, n2 = orc.tri_hit((0.25, 0.25, 1), (0, 0, -1), (0, 0, 0), (1, 0, 0), (0, 1, 0))
    assert t2 == 1.0 and n2[2] == 1.0
    assert orc.tri_hit((0.75, 0.75, -1), (0, 0, 1), (0, 0, 0), (1, 0, 0), (0, 1, 0)) is None
    # parallel ray: det == 0 -> miss
    assert orc.tri_hit((0.25, 0.25, 0), (1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0)) is None


def test_tie_break_smaller_id():
    """S:299 + P9: two coincident triangles ids 7 and 9 -> id 7 (also order-independent)."""
    rng = np.random.default_rng(1)
    verts = [rng.uniform(5, 6, size=(3, 3)) for _ in range(10)]   # far away decoys
    tri = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    verts[7] = tri
    verts[9] = tri
    v = np.concatenate(verts).astype(np.float32)
    idx = np.arange(30, dtype=np.int32).reshape(10, 3)
    sc = orc.OracleScene([di.Part(0, di.TRIS, verts=v, idx=idx)], 1)
    for brute in (True, False):
        t, i = sc.closest((0.25, 0.25, -1), (0, 0, 1), brute=brute)
        assert (t, i) == (1.0, 7)
    # reversed submission order: the coincident pair becomes ids 0 and 2 -> 0
    v2 = np.concatenate(verts[::-1]).astype(np.float32)
    sc2 = orc.OracleScene([di.Part(0, di.TRIS, verts=v2, idx=idx)], 1)
    assert sc2.closest((0.25, 0.25, -1), (0, 0, 1)) == (1.0, 0)


def _random_prims(seed, ntri=70, nsph=30):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1, 1, size=(ntri, 1, 3))
    v = (c + rng.uniform(-0.5, 0.5, size=(ntri, 3, 3))).astype(np.float32).reshape(-1, 3)
    idx = np.arange(3 * ntri, dtype=np.int32).reshape(-1, 3)
    sp = np.concatenate([rng.uniform(-1, 1, (nsph, 3)), rng.uniform(0.02, 0.2, (nsph, 1))], 1)
    return v, idx, sp.astype(np.float32)


def test_bvh_equals_brute_force():
    """P9 / S:290: oracle BVH closest (t,id) and any-hit == brute force on 10^4
    random rays over 100 random prims (70 tris + 30 spheres)."""
    v, idx, sp = _random_prims(3)
    sc = orc.OracleScene([di.Part(0, di.TRIS, verts=v, idx=idx),
                          di.Part(0, di.SPHERES, spheres=sp)], 1)
    rng = np.random.default_rng(4)
    o = rng.uniform(-1.5, 1.5, size=(10000, 3)).astype(np.float32)
    d = rng.standard_normal((10000, 3))
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    tm = rng.choice([np.inf, 0.5, 1.0], size=10000)
    nhit = 0
    for k in range(10000):
        a = sc.closest(o[k], d[k], tm[k], brute=True)
        b = sc.closest(o[k], d[k], tm[k], brute=False)
        assert a == b, (k, a, b)
        nhit += a[1] != 0xFFFFFFFF
        assert sc.any_hit(o[k], d[k], tm[k], True) == sc.any_hit(o[k], d[k], tm[k], False)
        assert sc.any_hit(o[k], d[k], tm[k]) == (a[1] != 0xFFFFFFFF)
    assert nhit > 1500


def test_slab_minnum_and_knife_edge():
    """P8 slab test: axis-parallel rays (inv=+-inf) and the knife-edge 0 <= -0 of H1."""
    ok, t0, t1 = orc.slab((-1, -1, -1), (1, 1, 1), (0, 0, -5), (0, 0, 1))
    assert ok and t0 == 4.0 and t1 == 6.0
    ok, _, _ = orc.slab((-1, -1, -1), (1, 1, 1), (2, 0, -5), (0, 0, 1))
    assert not ok
    z = np.float32(3) - np.float32(1e-4)
    ok, t0, t1 = orc.slab((-1, -1, z), (1, 1, np.float32(3) + np.float32(1e-4)),
                          (0.2, 0.2, z), (0, 0, -1))
    assert ok and t0 == 0.0 and t1 == 0.0
    ok, t0, _ = orc.slab((-1, -1, -1), (1, 1, 1), (0, 0, 0), (0, 0, 1))
    assert ok and t0 == 0.0  # origin inside: t0 clamps at 0


def test_camera_centre_and_fov():
    """P2 / S:324-325: centre pixel with jitter 0.5 -> d = w; fovy 90, aspect 1: the top
    pixel centre (sy=(H-0.5)/H) has elevation atan(1-1/H) (tan(45 deg)=1)."""
    W = H = 101
    cam = di.camera_basis((1, 2, 3), (1, 2, 13), (0, 1, 0), 90.0, W, H)
    fr = di.Frame(W=W, H=H, flags=1)
    o, d = orc.camera_ray(cam, fr, 50 * W + 50)
    assert np.allclose(d, [0, 0, 1], atol=2e-7) and np.array_equal(o, cam.E)
    _, d = orc.camera_ray(cam, fr, (H - 1) * W + 50)
    elev = math.atan2(d[1], d[2])
    assert abs(elev - math.atan(1 - 1 / H)) < 1e-6
    # bottom-left origin: pixel 0 looks down-right?  u = cross(w, up) = -x for w=+z
    _, d0 = orc.camera_ray(cam, fr, 0)
    assert d0[1] < 0 and d0[0] > 0
    # jittered: determinism and inside the pixel footprint
    fj = di.Frame(W=W, H=H, seed=7)
    a = orc.camera_ray(cam, fj, 1234, 3)[1]
    assert np.array_equal(a, orc.camera_ray(cam, fj, 1234, 3)[1])


def test_cosine_directions_distribution():
    """P7: cosine-weighted hemisphere (rejection + Duff et al. 2017 frame): unit length,
    upper hemisphere, E[cos]=2/3, E[cos^2]=1/2, tangential mean 0 -- for several normals
    including n.z<0 and n=-z (the frame's sign branch)."""
    for n in [(0, 0, 1), (0, 0, -1), (0.6, 0, -0.8), (0.48, 0.6, 0.64), (1, 0, 0)]:
        n = np.asarray(n, np.float32)
        ds = np.array([orc.cosine_dir(n, 7, p, 0, 0, 2, 0) for p in range(20000)])
        assert np.allclose(np.linalg.norm(ds, axis=1), 1, atol=1e-5)
        c = ds @ n
        assert (c >= -1e-6).all()
        assert abs(c.mean() - 2 / 3) < 0.01 and abs((c * c).mean() - 0.5) < 0.01
        tang = ds - c[:, None] * n
        assert np.linalg.norm(tang.mean(0)) < 0.02


def test_isotropic_directions():
    """P7 isotropic: unit length, mean 0, E[z^2] = 1/3."""
    ds = np.array([orc.iso_dir(7, p, 0, 0) for p in range(20000)])
    assert np.allclose(np.linalg.norm(ds, axis=1), 1, atol=1e-6)
    assert np.linalg.norm(ds.mean(0)) < 0.02 and abs((ds[:, 2] ** 2).mean() - 1 / 3) < 0.01


def _brick(vox, lo=(0, 0, 0), spacing=1.0, origin=(0, 0, 0), gd=None, tf=None):
    vox = np.asarray(vox, np.float32)
    nz, ny, nx = vox.shape
    hi = (lo[0] + nx - 1, lo[1] + ny - 1, lo[2] + nz - 1)
    return di.Part(0, di.BRICK, gdims=gd or (nx, ny, nz), origin=origin, spacing=(spacing,) * 3,
                   cell_lo=lo, cell_hi=hi, voxels=vox,
                   tf=tf if tf is not None else di.default_tf())


def test_trilinear_examples():
    """constant field -> constant; node -> node value; edge midpoint of 0,1 ->
    0.5.  P10: ownership is half-open [cell_lo, cell_hi)."""
    b = _brick(np.full((2, 2, 2), 5.0))
    assert orc.brick_sample(b, (0.3, 0.7, 0.2)) == 5.0
    rng = np.random.default_rng(0)
    vals = rng.uniform(0, 1, (3, 3, 3)).astype(np.float32)
    b = _brick(vals)
    for z in range(2):
        for y in range(2):
            for x in range(2):
                assert orc.brick_sample(b, (x, y, z)) == vals[z, y, x]
    e = np.zeros((2, 2, 2), np.float32)
    e[0, 0, 1] = 1.0
    assert orc.brick_sample(_brick(e), (0.5, 0, 0)) == 0.5
    # x-fastest storage: value along y
    e = np.zeros((2, 2, 2), np.float32)
    e[0, 1, 0] = 1.0
    assert orc.brick_sample(_brick(e), (0, 0.25, 0)) == 0.25
    assert orc.brick_sample(_brick(e), (1.0, 0, 0)) is None        # g == cell_hi: not owned
    assert orc.brick_sample(_brick(e), (-1e-3, 0, 0)) is None
    # brick offset in a global grid: global coordinates with the global origin
    b = _brick(vals, lo=(4, 4, 4), spacing=0.5, origin=(-1, -1, -1), gd=(9, 9, 9))
    assert orc.brick_sample(b, (1.0, 1.0, 1.0)) == vals[0, 0, 0]


def test_transfer_function_examples():
    """clamp below/above the domain; linear interpolation; alpha*densityScale
    clamped at 1."""
    s = np.arange(256, dtype=np.float64) / 255
    tf = np.stack([s, s, s, s], 1).astype(np.float32)
    assert np.array_equal(orc.tf_eval(tf, 0, 1, 1, -3), tf[0])
    assert np.allclose(orc.tf_eval(tf, 0, 1, 1, 7), tf[255])
    r = orc.tf_eval(tf, 0, 1, 1, 0.5)
    assert np.allclose(r, 0.5, atol=1e-6)
    r = orc.tf_eval(tf, 0, 1, 3.0, 0.5)
    assert np.allclose(r[:3], 0.5, atol=1e-6) and r[3] == 1.0
    r = orc.tf_eval(tf, 0, 1, 0.5, 0.5)
    assert abs(r[3] - 0.25) < 1e-6


def test_bvh_equals_brute_force_tiny_clustered_spheres():
    """P9 on the configs[3] sphere family (dense Gaussian clusters of r ~ 0.003 spheres, rays
    from inside and outside the clusters): oracle BVH closest/any == brute force.  This pins
    reading R-SPHERE: with the b^2-(|f|^2-r^2) discriminant, rounding let small distant
    spheres report hits outside their own bounding box, which no BVH can find."""
    sph = di.sphere_clusters(6, 1500, 0.05, 0.002, 0.004, seed=5)
    sc = orc.OracleScene([di.Part(0, di.SPHERES, spheres=sph)], 1)
    rng = np.random.default_rng(9)
    centres = sph[:, :3].astype(np.float64)
    mism = 0
    for k in range(6000):
        if k % 2 == 0:   # from far away toward a random sphere
            o = rng.uniform(-2.5, 2.5, 3)
            tgt = centres[rng.integers(len(centres))] + rng.normal(0, 0.004, 3)
        else:            # from inside a cluster
            o = centres[rng.integers(len(centres))] + rng.normal(0, 0.01, 3)
            tgt = o + rng.normal(0, 1, 3)
        d = (tgt - o) / np.linalg.norm(tgt - o)
        o, d = o.astype(np.float32), d.astype(np.float32)
        tm = np.inf if k % 3 else 0.1
        a = sc.closest(o, d, tm, brute=True)
        b = sc.closest(o, d, tm)
        mism += a != b
        assert sc.any_hit(o, d, tm, True) == sc.any_hit(o, d, tm)
    assert mism == 0


def test_sphere_far_tangent_is_box_consistent():
    """R-SPHERE: a reported hit lies within the sphere's box (up to float rounding) even for
    a tiny sphere far from the ray origin."""
    c = np.array([1.7, -0.3, 0.9], np.float32)
    r = np.float32(0.003)
    rng = np.random.default_rng(2)
    for _ in range(4000):
        o = rng.uniform(-2, 2, 3).astype(np.float32)
        tgt = c + rng.uniform(-1.2, 1.2, 3) * r
        d = ((tgt - o) / np.linalg.norm(tgt - o)).astype(np.float32)
        h = orc.sphere_hit(o, d, c, float(r))
        if h is None:
            continue
        p = o.astype(np.float64) + h[0] * d.astype(np.float64)
        assert np.all(np.abs(p - c) <= r * (1 + 1e-3) + 1e-6), (p - c, r)


def _plain_p3_hits(o, d, v0, e1, e2):
    """Input selection only: P3 in binary32 WITHOUT the R-DEGEN rule (edges as given)."""
    f = np.float32

    def cross(a, b):
        return np.array([a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2],
                         a[0] * b[1] - a[1] * b[0]], f)

    def dot(a, b):
        return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]

    pv = cross(d, e2)
    det = dot(e1, pv)
    if det == 0:
        return False
    inv = f(1) / det
    tv = o - v0
    uu = dot(tv, pv) * inv
    if uu < 0 or uu > 1:
        return False
    qv = cross(tv, e1)
    vv = dot(d, qv) * inv
    if vv < 0 or uu + vv > 1:
        return False
    return dot(e2, qv) * inv > 0


def _collinear_hits(n_want=20, seed=0):
    """Rays aimed at points of exactly-collinear triangles (binary32 cross(e1,e2) == 0)
    that plain P3 arithmetic reports as hit (det != 0 by rounding)."""
    rng = np.random.default_rng(seed)
    out = []
    f = np.float32
    with np.errstate(all="ignore"):
        while len(out) < n_want:
            v0 = rng.uniform(-1, 1, 3).astype(f)
            e = rng.uniform(-1, 1, 3).astype(f)
            v1 = (v0 + e).astype(f)
            v2 = (v0 + f(rng.uniform(0.2, 2.0)) * e).astype(f)
            e1, e2 = v1 - v0, v2 - v0
            ng = np.array([e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                           e1[0] * e2[1] - e1[1] * e2[0]], f)
            if np.any(ng != 0):
                continue
            pt = (v0 + f(0.3) * (v1 - v0)).astype(f)
            o = (pt + rng.uniform(-2, 2, 3)).astype(f)
            d = (pt - o).astype(np.float64)
            d = (d / np.linalg.norm(d)).astype(f)
            if _plain_p3_hits(o, d, v0, e1, e2):
                out.append((o, d, v0, v1, v2))
    return out


def test_zero_area_triangle_never_hit():
    """Reading R-DEGEN: a triangle whose binary32 cross(e1, e2) is the zero vector has no area
    and no normal (the P3 normal would be 0/0); it is never hit -- neither by the single
    intersection test nor inside a rendered world (where such triangles stand in the ray's
    way of a real one behind them)."""
    cases = _collinear_hits()
    for o, d, v0, v1, v2 in cases:
        assert orc.tri_hit(o, d, v0, v1, v2) is None
    # a world of only those triangles + a big quad behind them: every ray hits the quad
    for o, d, v0, v1, v2 in cases[:5]:
        c = (o + 50 * d.astype(np.float64)).astype(np.float32)
        u = np.cross(d, [0.3, 0.5, 0.8]); u /= np.linalg.norm(u)
        w = np.cross(d, u)
        quad = [c + 40 * (a * u + b * w) for a, b in ((-1, -1), (1, -1), (1, 1), (-1, 1))]
        qv, qi = di.quad_tris(quad)
        parts = [di.Part(0, di.TRIS, albedo=(1, 1, 1), verts=di.f32([v0, v1, v2]),
                         idx=np.array([[0, 1, 2]], np.int32)),
                 di.Part(0, di.TRIS, albedo=(1, 1, 1), verts=qv, idx=qi)]
        sc = orc.OracleScene(parts, 1)
        t, i = sc.closest(o, d)
        assert i in (1, 2) and 49 < t < 51, (t, i)
        assert np.isfinite(t)


def test_invalid_primitives_rejected():
    """dpr.h: coordinates must be finite and sphere radii > 0; the oracle refuses such a
    world as the GPU path does (DPR_ERR_INVALID_ARG)."""
    ok = di.Part(0, di.SPHERES, spheres=di.f32([[0, 0, 0, 1]]))
    orc.OracleScene([ok], 1)
    for sph in ([0, 0, 0, 0], [0, 0, 0, -1], [np.nan, 0, 0, 1], [0, 0, 0, np.inf]):
        with pytest.raises(ValueError):
            orc.OracleScene([di.Part(0, di.SPHERES, spheres=di.f32([sph]))], 1)
    with pytest.raises(ValueError):
        orc.OracleScene([di.Part(0, di.TRIS, verts=di.f32([(0, 0, 0), (1, np.inf, 0), (0, 1, 0)]),
                                 idx=np.array([[0, 1, 2]], np.int32))], 1)
