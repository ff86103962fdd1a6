"""Oracle pins, part 5: the P1 counter / purpose layout of every RNG call site.

SURVEY 8(c).2 P1 fixes, for Philox4x32-10 (itself pinned by the Random123 KATs in
test_oracle_primitives.py), key = (seed lo, seed hi) and counter = (p, s, (depth<<8) |
purpose, sub) with:
  0 camera jitter   sub 0, x0 -> jx, x1 -> jy
  2 AO ray k        sub = (k<<4) | attempt
  3 bounce          sub = attempt
  4/5/6 volume sample i of a path / shadow / AO-k ray: sub = (AO: k<<24) | (i>>2), lane i&3
Each test below re-derives the draws from `oracle.philox` (KAT-verified) by that table and
compares them with what the oracle's renderer actually consumes -- through the single-call
exports of the renderer's own call sites, and through whole renders whose event codes /
occlusion bits reveal the draws (a direction's sign, the first colliding volume sample).
`tools/oracle_mutations.py` records that each test fails under a one-field mutation of the
layout (profiles/r02_oracle_mutations.json).
"""
import numpy as np
import pytest

import dpr_inputs as di
import oracle as orc

SEEDS = [7, 0x9E3779B97F4A7C15]  # the pinned frame seed, and one with high key bits set
F32 = np.float32


def draws(seed, p, s, depth, purpose, sub):
    """P1: Philox4x32-10 at counter (p, s, (depth<<8)|purpose, sub), key (lo, hi)."""
    return orc.philox([p, s, (depth << 8) | purpose, sub],
                      [seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF])


def u(x):
    """P1 to-float: (x>>8) * 2^-24, exact in binary32."""
    return F32(x >> 8) * F32(2.0 ** -24)


def disc_draw(seed, p, s, depth, purpose, subhi):
    """P7 rejection: the first attempt a < 16 with r2 < 1 of (2u0-1, 2u1-1); None if none."""
    for a in range(16):
        x = draws(seed, p, s, depth, purpose, subhi | a)
        vx, vy = F32(2) * u(x[0]) - F32(1), F32(2) * u(x[1]) - F32(1)
        r2 = vx * vx + vy * vy
        if r2 < F32(1):
            return vx, vy, np.sqrt(F32(1) - r2)
    return None


@pytest.mark.parametrize("seed", SEEDS)
def test_camera_jitter_counter(seed):
    """Purpose 0: jx = u(x0), jy = u(x1) of counter (p, s, 0, 0).  With E = 0, L = (0,0,1),
    U = (1,0,0), V = (0,1,0) the P2 ray direction is (sx, sy, 1)/len, so sx = d.x/d.z =
    (x + jx)/W recovers the jitter to ~1e-6 (a wrong counter field gives an unrelated
    value)."""
    W = H = 8
    cam = di.Camera(E=di.f32((0, 0, 0)), L=di.f32((0, 0, 1)), U=di.f32((1, 0, 0)),
                    V=di.f32((0, 1, 0)))
    fr = di.Frame(W=W, H=H, spp=4, seed=seed, flags=0)
    for p in range(W * H):
        x, y = p % W, p // W
        for s in range(4):
            _, d = orc.camera_ray(cam, fr, p, s)
            d = d.astype(np.float64)
            jx, jy = d[0] / d[2] * W - x, d[1] / d[2] * H - y
            r = draws(seed, p, s, 0, 0, 0)
            assert abs(jx - float(u(r[0]))) < 1e-5, (p, s, jx, float(u(r[0])))
            assert abs(jy - float(u(r[1]))) < 1e-5, (p, s, jy, float(u(r[1])))


@pytest.mark.parametrize("seed", SEEDS)
def test_ao_and_bounce_counters_exports(seed):
    """Purposes 2 and 3 at the renderer's call sites (ao_dir / bounce_dir).  For n = +z the
    Duff et al. frame is the identity (t1 = (1,-0,-0), t2 = (-0,1,-0)), so the direction is
    exactly (2u0-1, 2u1-1, sqrt(1-r2)) of the first accepted attempt."""
    n = (0.0, 0.0, 1.0)
    for p in (0, 1, 77, 123456):
        for s in (0, 3):
            for depth in (0, 1, 5):
                for k in range(4):
                    want = disc_draw(seed, p, s, depth, 2, k << 4)
                    got = orc.ao_dir(n, seed, p, s, depth, k)
                    assert np.array_equal(got, np.array(want, F32)), (p, s, depth, k, got, want)
                want = disc_draw(seed, p, s, depth, 3, 0)
                assert np.array_equal(orc.bounce_dir(n, seed, p, s, depth), np.array(want, F32))


@pytest.mark.parametrize("seed", SEEDS)
def test_volume_counters_export(seed):
    """Purposes 4/5/6: u_i = lane i&3 of counter sub (AO k: k<<24) | (i>>2)."""
    for kind, purpose in ((0, 4), (1, 5), (2, 6)):
        for k in ((0,) if kind < 2 else (0, 1, 5)):
            for p, s, depth in ((0, 0, 0), (99, 2, 1), (4097, 15, 3)):
                for i in list(range(12)) + [1023, 4096 + 3]:
                    sub = (k << 24 if kind == 2 else 0) | (i >> 2)
                    want = u(draws(seed, p, s, depth, purpose, sub)[i & 3])
                    assert orc.vol_u(seed, p, s, depth, kind, k, i) == float(want), (kind, k, p, s, i)


def _ao_wall_scene(spp, K, max_depth):
    """Eye (0,0,5) looking straight down at the ground z=0 (normal +z at the hit (0,0,0));
    a wall x = 0.01 (id 2, 3) stands next to the hit point.  A ray leaving (0,0,1e-4)
    upward hits the wall iff its direction has x > 0."""
    g, gi = di.quad_tris([(-5, -5, 0), (5, -5, 0), (5, 5, 0), (-5, 5, 0)])
    w, wi = di.quad_tris([(0.01, -1e4, -1), (0.01, 1e4, -1), (0.01, 1e4, 1e6), (0.01, -1e4, 1e6)])
    parts = [di.Part(0, di.TRIS, albedo=(0.5, 0.5, 0.5), verts=g, idx=gi),
             di.Part(0, di.TRIS, albedo=(0.5, 0.5, 0.5), verts=w, idx=wi)]
    cam = di.camera_basis((0, 0, 5), (0, 0, 0), (0, 1, 0), 10.0, 1, 1)
    fr = di.Frame(W=1, H=1, spp=spp, spp_batch=spp, max_depth=max_depth, ao_k=K,
                  ao_radius=1e30, light_dir=(0, 0, 1), E=(0, 0, 0), A=(1, 1, 1), seed=7,
                  flags=1)
    return parts, cam, fr


def test_ao_counter_through_render():
    """AO ray k of sample s (depth 0) is unoccluded (occl bit 1+k) iff the x of its first
    accepted disc draw (purpose 2, sub (k<<4)|a) is <= 0: the wall takes x > 0."""
    spp, K = 64, 4
    parts, cam, fr = _ao_wall_scene(spp, K, 1)
    r = orc.render(orc.OracleScene(parts, 1), cam, fr)
    assert (r.events[:, 0, 0] == 2).all() or (r.events[:, 0, 0] == 3).all()
    for s in range(spp):
        for k in range(K):
            vx = disc_draw(7, 0, s, 0, 2, k << 4)[0]
            assert bool((r.occl[s, 0, 0] >> (1 + k)) & 1) == (vx <= 0), (s, k)
    free = sum(bin(int(r.occl[s, 0, 0]) >> 1).count("1") for s in range(spp))
    assert 0 < free < spp * K  # both outcomes occur


def test_bounce_counter_through_render():
    """The bounce of sample s (depth 0 -> event at depth 1) hits the wall (ids 2/3) iff the x
    of its first accepted disc draw (purpose 3, sub a) is > 0, else it escapes (event 1)."""
    spp = 64
    parts, cam, fr = _ao_wall_scene(spp, 0, 2)
    r = orc.render(orc.OracleScene(parts, 1), cam, fr)
    hits = 0
    for s in range(spp):
        vx = disc_draw(7, 0, s, 0, 3, 0)[0]
        ev = int(r.events[s, 1, 0])
        assert (ev in (4, 5)) == (vx > 0) and (ev == 1) == (vx <= 0), (s, ev, vx)
        hits += vx > 0
    assert 0 < hits < spp


def _const_brick(gdims, origin, h, alpha, value=0.5):
    tf = np.zeros((256, 4), np.float32)
    tf[:, :3] = (0.3, 0.6, 0.9)
    tf[:, 3] = alpha
    nx, ny, nz = gdims
    return di.Part(0, di.BRICK, gdims=gdims, origin=origin, spacing=(h, h, h),
                   cell_lo=(0, 0, 0), cell_hi=(nx - 1, ny - 1, nz - 1),
                   voxels=np.full((nz, ny, nx), value, np.float32), tf=tf)


def test_volume_path_counter_through_render():
    """Purpose 4 (path ray): with a constant opacity alpha every owned sample collides iff
    u_i < alpha, so the event is 0x80000000 | (first i >= i0 with u_i < alpha), where i0 is
    the first owned sample (the event of the alpha = 1 render)."""
    G, h = 33, float(np.float32(2.0 / 32))
    cam = di.camera_basis((0.05, 0.03, -3), (0.05, 0.03, 0), (0, 1, 0), 10.0, 1, 1)
    spp = 64

    def run(alpha):
        fr = di.Frame(W=1, H=1, spp=spp, spp_batch=spp, max_depth=1, dt=h, seed=7, flags=1)
        parts = [_const_brick((G, G, G), (-1, -1, -1), h, alpha)]
        return orc.render(orc.OracleScene(parts, 1), cam, fr)

    i0 = run(1.0).events[:, 0, 0]
    assert (i0 == i0[0]).all() and (i0[0] & 0x80000000)
    i0 = int(i0[0] & 0x7FFFFFFF)
    alpha = np.float32(0.3)
    ev = run(float(alpha)).events[:, 0, 0]
    for s in range(spp):
        i = i0
        while not u(draws(7, 0, s, 0, 4, i >> 2)[i & 3]) < alpha:
            i += 1
        assert int(ev[s]) == (0x80000000 | i), (s, hex(int(ev[s])), i)


def test_volume_shadow_counter_through_render():
    """Purpose 5 (shadow ray): the ground point (0,0,0) is lit from +z through a constant
    layer whose owned samples along the shadow ray are exactly i = 0..5 (grid z = i + 0.301,
    owned: 0 <= g < 6), so the shadow bit is set iff u_i >= alpha for i = 0..5 (counter
    sub i>>2 spans two Philox blocks).  The primary comes in at a grazing angle below the
    layer."""
    h = 0.1
    layer = _const_brick((5, 5, 7), (-0.2, -0.2, 0.02), h, 0.15)
    g, gi = di.quad_tris([(-5, -5, 0), (5, -5, 0), (5, 5, 0), (-5, 5, 0)])
    parts = [di.Part(0, di.TRIS, albedo=(1, 1, 1), verts=g, idx=gi), layer]
    cam = di.camera_basis((3, 0, 0.05), (0, 0, 0), (0, 0, 1), 1.0, 1, 1)
    spp = 128
    fr = di.Frame(W=1, H=1, spp=spp, spp_batch=spp, max_depth=1, ao_k=0, light_dir=(0, 0, 1),
                  E=(1, 1, 1), dt=float(np.float32(h)), seed=7, flags=1)
    r = orc.render(orc.OracleScene(parts, 1), cam, fr)
    assert (r.events[:, 0, 0] < 0x80000000).all() and (r.events[:, 0, 0] >= 2).all()
    alpha = np.float32(0.15)
    lit = 0
    for s in range(spp):
        free = all(not u(draws(7, 0, s, 0, 5, i >> 2)[i & 3]) < alpha for i in range(6))
        assert bool(r.occl[s, 0, 0] & 1) == free, s
        lit += free
    assert 0 < lit < spp
