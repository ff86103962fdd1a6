"""Oracle pins for delta tracking (NEXT f4; readings R-DELTA, R-LOG): Woodcock
tracking with one global majorant.  The pins are facts about the estimator, not re-typings:
  * the pinned log agrees with libm's double log to < 1 ulp over (2^-24, 1];
  * Beer-Lambert: the probability of a collision over a chord of length L in a medium of
    extinction mu = alpha/dt is 1 - exp(-mu L), with a tight majorant AND with a loose one
    (null collisions must not bias it), and the collision depth is exponential;
  * binary shadow transmittance exp(-mu L);
  * partition independence: bricks over several ranks render bit-identically to the union.
"""
import math
import struct

import numpy as np
import pytest

import dpr_inputs as di
import oracle as orc

DELTA = 16


def _ulp(y):
    b = struct.unpack("<I", struct.pack("<f", abs(y)))[0]
    return struct.unpack("<f", struct.pack("<I", b + 1))[0] - abs(float(np.float32(y)))


def test_pinned_log_accuracy():
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(0, 1, 20000), 2.0 ** -rng.uniform(0, 24, 20000),
                         [1.0, 0.5, 0.25, 2.0 ** -24, 0.70710677, 0.70710683, 0.9999999, 0.99999994]])
    xs = xs.astype(np.float32)
    xs = xs[xs > 0]
    worst = 0.0
    for x in xs:
        r, ref = orc.pln(float(x)), math.log(float(x))
        if ref == 0.0:
            assert r == 0.0
            continue
        worst = max(worst, abs(r - ref) / _ulp(ref))
    assert worst < 1.0, worst
    # exact powers of two: e*ln2 to within one ulp; monotone on a fine sweep
    for e in range(1, 24):
        assert abs(orc.pln(2.0 ** -e) + e * math.log(2)) <= _ulp(e * math.log(2))
    sweep = np.float32(np.linspace(0.6, 0.8, 3001))
    vals = [orc.pln(float(x)) for x in sweep]
    assert all(a <= b for a, b in zip(vals, vals[1:]))


def _volume(G, alpha_field, tf_alpha, nbricks=1, nranks=1):
    """Constant density 0.5 in a G^3 grid over [-1,1]^3; the TF maps density s in [0,1]
    linearly from tf_alpha[0] (s=0) to tf_alpha[1] (s=1) -> alpha(0.5) = alpha_field."""
    tf = np.zeros((256, 4), np.float32)
    tf[:, :3] = (0.2, 0.5, 0.8)
    tf[:, 3] = np.linspace(tf_alpha[0], tf_alpha[1], 256, dtype=np.float32)
    h = np.float32(2.0 / (G - 1))
    parts = []
    for r, (lo, hi) in enumerate(di.brick_boxes((G - 1,) * 3, nbricks)):
        nx, ny, nz = hi[0] - lo[0] + 1, hi[1] - lo[1] + 1, hi[2] - lo[2] + 1
        parts.append(di.Part(r % nranks, di.BRICK, gdims=(G,) * 3, origin=(-1, -1, -1),
                             spacing=(float(h),) * 3, cell_lo=lo, cell_hi=hi,
                             voxels=np.full((nz, ny, nx), 0.5, np.float32), tf=tf))
    a = float(orc.tf_eval(tf, 0.0, 1.0, 1.0, 0.5)[3])
    assert abs(a - alpha_field) < 2e-3
    return parts, a


@pytest.mark.parametrize("loose", [False, True])
def test_collision_probability_is_beer_lambert(loose):
    """Rays along +z through the 2-unit-thick cube: P(collision) = 1 - exp(-alpha/dt * 2).
    loose=True uses a TF whose peak (unused by the constant field) is 4x the field's alpha,
    so 3/4 of the tentative collisions are null collisions."""
    alpha, dt = 0.01, 0.02
    tfa = (alpha, alpha) if not loose else (-2 * alpha, 4 * alpha)  # alpha(0.5) = alpha either way
    parts, a = _volume(9, alpha, tfa)
    mu = a / dt
    cam = di.camera_basis((0.013, 0.007, -3), (0.013, 0.007, 0), (0, 1, 0), 0.5, 1, 1)
    spp = 8000
    fr = di.Frame(W=1, H=1, spp=spp, spp_batch=spp, max_depth=1, ao_k=0, dt=dt, E=(0, 0, 0),
                  flags=1 | DELTA)
    r = orc.render(orc.OracleScene(parts, 1), cam, fr)
    ev = r.events[:, 0, 0]
    hit = (ev & 0x80000000) != 0
    o, d = orc.camera_ray(cam, fr, 0)
    L = 2.0 / float(d[2])
    p = 1 - math.exp(-mu * L)
    assert abs(hit.mean() - p) < 4 * math.sqrt(p * (1 - p) / spp), (hit.mean(), p)
    # with a loose majorant the first real collision is rarely the first tentative point
    k = ev[hit] & 0x7FFFFFFF
    if loose:
        assert (k > 0).mean() > 0.5
    else:
        assert (k == 0).all()


def test_collision_depth_is_exponential():
    """The first-collision depth x = t - t_entry in a homogeneous medium is Exp(mu), with
    null collisions in play (loose majorant): empirical CDF at several depths vs
    1 - exp(-mu x).  One sample per pixel; the depth buffer of the local render gives t."""
    alpha, dt = 0.02, 0.02
    parts, a = _volume(9, alpha, (-alpha, 3 * alpha))
    mu = a / dt
    W = H = 64
    cam = di.camera_basis((0, 0, -3), (0, 0, 0), (0, 1, 0), 8.0, W, H)
    fr = di.Frame(W=W, H=H, spp=1, spp_batch=1, max_depth=1, ao_k=0, dt=dt, E=(0, 0, 0),
                  flags=1 | DELTA)
    _, depth = orc.render_local_fragments(parts, 0, cam, fr)
    xs, chords = [], []
    for pix in range(W * H):
        o, d = (v.astype(np.float64) for v in orc.camera_ray(cam, fr, pix))
        t0, t1 = (-1 - o[2]) / d[2], (1 - o[2]) / d[2]
        xs.append(depth[pix] - t0 if np.isfinite(depth[pix]) else np.inf)
        chords.append(t1 - t0)
    xs = np.array(xs)
    n = len(xs)
    assert min(chords) > 1.99
    for q in (0.1, 0.25, 0.5, 1.0, 1.9):
        p = 1 - math.exp(-mu * q)
        emp = (xs < q).mean()
        assert abs(emp - p) < 4 * math.sqrt(p * (1 - p) / n) + 1e-3, (q, emp, p)


def test_shadow_transmittance_is_beer_lambert():
    """Binary shadows through the homogeneous cube: P(unoccluded) = exp(-mu L)."""
    alpha, dt = 0.015, 0.02
    parts, a = _volume(9, alpha, (0.0, 2 * alpha))
    mu = a / dt
    plane = di.Part(0, di.TRIS, albedo=(1, 1, 1),
                    verts=di.f32([[-3, -1.5, -3], [3, -1.5, -3], [3, -1.5, 3], [-3, -1.5, 3]]),
                    idx=np.array([[0, 1, 2], [0, 2, 3]], np.int32))
    cam = di.camera_basis((0.01, -1.0, -3.0), (0.01, -1.5, 0.0), (0, 1, 0), 1.0, 1, 1)
    spp = 4000
    fr = di.Frame(W=1, H=1, spp=spp, spp_batch=spp, max_depth=1, ao_k=0, dt=dt,
                  light_dir=(0, 1, 0), E=(1, 1, 1), flags=1 | DELTA)
    r = orc.render(orc.OracleScene(parts + [plane], 1), cam, fr)
    ev = r.events[:, 0, 0]
    surf = (ev & 0x80000000) == 0
    assert surf.mean() > 0.99          # the primary passes under the cube
    lit = (r.occl[:, 0, 0] & 1) != 0
    p = math.exp(-mu * 2.0)            # the shadow ray crosses the full 2-unit height
    n = int(surf.sum())
    assert abs(lit[surf].mean() - p) < 4 * math.sqrt(p * (1 - p) / n), (lit[surf].mean(), p)


@pytest.mark.parametrize("nbricks,nranks", [(4, 2), (8, 4), (3, 3)])
def test_delta_tracking_partition_independence(nbricks, nranks):
    """Bricks over ranks (routing simulator) == one rank with all bricks (union renderer):
    events, occlusion bits, pixels identical (P:657-659 invariant under R-DELTA)."""
    G = 25
    field = di.volume_field(G)
    tf = di.default_tf(alpha_max=0.3, s0=0.2)
    h = np.float32(2.0 / (G - 1))
    parts = []
    for r, (lo, hi) in enumerate(di.brick_boxes((G - 1,) * 3, nbricks)):
        vox = field[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
        parts.append(di.Part(r % nranks, di.BRICK, gdims=(G,) * 3, origin=(-1, -1, -1),
                             spacing=(float(h),) * 3, cell_lo=lo, cell_hi=hi,
                             voxels=np.ascontiguousarray(vox), tf=tf))
    W = H = 20
    cam = di.camera_basis((0.3, 1.5, -3.0), (0, -0.2, 0), (0, 1, 0), 50.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=1, max_depth=2, ao_k=1, ao_radius=0.3, dt=float(h),
                  light_dir=di.f32(di.normalize((0.2, 1, 0.1))), E=(1, 1, 1), A=(0.2, 0.2, 0.2),
                  flags=DELTA)
    dp = orc.render(orc.OracleScene(parts, nranks), cam, fr, dp=True)
    u = orc.render(orc.OracleScene(di.union_parts(parts), 1), cam, fr)
    assert np.array_equal(dp.events, u.events) and np.array_equal(dp.occl, u.occl)
    assert np.allclose(dp.rgba, u.rgba, atol=1e-12, rtol=0)
    assert ((u.events & 0x80000000) != 0).sum() > 50
