"""Oracle pins for the thin-lens camera ("rendered with depth of field"; DESIGN.md
reading R-DOF).  Each pin is an external fact about a thin lens, not a re-typing of the
oracle's formula:
  * every ray of a sample passes through the pinhole ray's point on the focal plane;
  * ray origins lie on the lens disc (radius r, in the image-plane axes, centred on E) and
    are uniformly distributed there (E[rho^2] = r^2/2, P(rho < r/2) = 1/4, zero mean);
  * a surface in the focal plane renders exactly as with the pinhole camera;
  * out-of-focus geometry is blurred by the circle of confusion r*|fd - z|/fd: the radial
    coverage profile of a sphere matches an independent float64 Monte Carlo thin-lens model.
"""
import dataclasses
import math

import numpy as np

import dpr_inputs as di
import oracle as orc


def _cam(W=64, H=64, fovy=20.0, r=0.2, fd=8.0, pos=(0, 0, -4)):
    c = di.camera_basis(pos, (0, 0, 0), (0, 1, 0), fovy, W, H)
    return dataclasses.replace(c, lens_radius=r, focus_dist=fd)


def _q(cam, x, y, W, H, jx=0.5, jy=0.5):
    sx, sy = (x + jx) / W, (y + jy) / H
    return cam.L.astype(np.float64) + sx * cam.U.astype(np.float64) + sy * cam.V.astype(np.float64)


def test_lens_zero_is_pinhole():
    W = H = 16
    cam = _cam(W, H, r=0.0, fd=3.0)
    pin = _cam(W, H, r=0.0, fd=0.0)
    fr = di.Frame(W=W, H=H, spp=2)
    for p in range(0, W * H, 7):
        for s in range(2):
            a, b = orc.camera_ray(cam, fr, p, s), orc.camera_ray(pin, fr, p, s)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_rays_pass_through_focal_point_and_start_on_lens():
    W, H = 32, 24
    cam = _cam(W, H, fovy=35.0, r=0.3, fd=5.0, pos=(0.5, 1.0, -4))
    fr = di.Frame(W=W, H=H, spp=8, flags=1)   # jitter-centre: q known in closed form
    E = cam.E.astype(np.float64)
    w = di.normalize(np.array([0, 0, 0]) - np.array([0.5, 1.0, -4]))
    for p in range(0, W * H, 5):
        x, y = p % W, p // W
        F = E + cam.focus_dist * _q(cam, x, y, W, H)
        assert abs((F - E) @ w - cam.focus_dist) < 1e-5          # F is on the focal plane
        for s in range(8):
            o, d = (v.astype(np.float64) for v in orc.camera_ray(cam, fr, p, s))
            assert abs(np.linalg.norm(d) - 1) < 1e-6
            off = o - E
            assert np.linalg.norm(off) <= cam.lens_radius * (1 + 1e-6)
            assert abs(off @ w) < 1e-6                               # lens plane is normal to w
            v = F - o
            dist = np.linalg.norm(v - (v @ d) * d)                   # F's distance from the ray
            assert dist < 2e-6 * np.linalg.norm(v), (p, s, dist)


def test_lens_samples_uniform_on_disc():
    W = H = 64
    r = 0.5
    cam = _cam(W, H, r=r, fd=4.0)
    fr = di.Frame(W=W, H=H, spp=4)
    E = cam.E.astype(np.float64)
    u = cam.U.astype(np.float64) / np.linalg.norm(cam.U)
    v = cam.V.astype(np.float64) / np.linalg.norm(cam.V)
    pts = []
    for p in range(W * H):
        for s in range(4):
            o, _ = orc.camera_ray(cam, fr, p, s)
            off = o.astype(np.float64) - E
            pts.append((off @ u / r, off @ v / r))
    pts = np.array(pts)
    rho2 = (pts ** 2).sum(1)
    n = len(pts)
    assert rho2.max() <= 1 + 1e-5
    assert abs(rho2.mean() - 0.5) < 4 * math.sqrt(1 / 12 / n)        # square: 2/3; uniform disc: 1/2
    assert abs((rho2 < 0.25).mean() - 0.25) < 4 * math.sqrt(0.1875 / n)
    assert np.abs(pts.mean(0)).max() < 4 * math.sqrt(0.25 / n)
    # the angle is uniform too (quadrant counts)
    q = np.bincount((pts[:, 0] > 0) * 2 + (pts[:, 1] > 0), minlength=4) / n
    assert np.abs(q - 0.25).max() < 4 * math.sqrt(0.1875 / n)


def _checker_plane(z=0.0, cells=8, ext=2.0):
    parts = []
    h = 2 * ext / cells
    for i in range(cells):
        for j in range(cells):
            x0, y0 = -ext + i * h, -ext + j * h
            v, idx = di.quad_tris([(x0, y0, z), (x0 + h, y0, z), (x0 + h, y0 + h, z), (x0, y0 + h, z)])
            rho = (0.9, 0.2, 0.1) if (i + j) % 2 else (0.1, 0.3, 0.9)
            parts.append(di.Part(0, di.TRIS, albedo=rho, verts=v, idx=idx))
    return parts


def test_in_focus_plane_renders_as_pinhole():
    """A checkerboard lying in the focal plane: every lens ray of a sample meets the plane
    at the pinhole ray's hit point, so the image equals the pinhole image."""
    W = H = 48
    parts = _checker_plane()
    pin = _cam(W, H, fovy=40.0, r=0.0, fd=0.0)
    dof = _cam(W, H, fovy=40.0, r=0.3, fd=4.0)
    fr = di.Frame(W=W, H=H, spp=4, max_depth=1, ao_k=0, light_dir=di.f32((0, 0, -1)),
                  E=(1, 1, 1), A=(0, 0, 0), B=(0, 0, 0), flags=1)
    a = orc.render(orc.OracleScene(parts, 1), pin, fr)
    b = orc.render(orc.OracleScene(parts, 1), dof, fr)
    assert np.abs(a.rgba - b.rgba).max() < 1e-6
    # out of focus (fd = 2) the checker edges blur: many pixels change
    c = orc.render(orc.OracleScene(parts, 1), dataclasses.replace(dof, focus_dist=2.0), fr)
    assert (np.abs(a.rgba - c.rgba).max(1) > 0.05).mean() > 0.2


def _profile(cov, W, H, nb):
    yy, xx = np.mgrid[0:H, 0:W]
    rad = np.hypot(xx + 0.5 - W / 2, yy + 0.5 - H / 2).ravel()
    b = np.minimum((rad / 2).astype(int), nb - 1)
    return np.bincount(b, cov, nb) / np.maximum(np.bincount(b, None, nb), 1)


def test_defocus_blur_matches_thin_lens_model():
    """Coverage of a sphere (R=0.2, 4 units away) with the focal plane at 8 and lens radius
    0.2: circle of confusion radius 0.2*4/8 = 0.1 at the sphere -> a ~9-pixel soft edge.
    The oracle's radial profile equals an independent float64 Monte Carlo thin-lens model
    (polar lens sampling, analytic ray-sphere) and the pinhole edge is sharp."""
    W = H = 64
    R = 0.2
    sph = di.Part(0, di.SPHERES, albedo=(1, 1, 1), spheres=di.f32([[0, 0, 0, R]]))
    fr = di.Frame(W=W, H=H, spp=64, spp_batch=64, max_depth=1, ao_k=0, seed=11)
    dof = _cam(W, H, r=0.2, fd=8.0)
    got = orc.render(orc.OracleScene([sph], 1), dof, fr).rgba[:, 3]
    pin = orc.render(orc.OracleScene([sph], 1), _cam(W, H, r=0.0, fd=0.0), fr).rgba[:, 3]

    rng = np.random.default_rng(0)
    M = 256
    E = dof.E.astype(np.float64)
    u = dof.U.astype(np.float64) / np.linalg.norm(dof.U)
    v = dof.V.astype(np.float64) / np.linalg.norm(dof.V)
    ref = np.zeros(W * H)
    yy, xx = np.mgrid[0:H, 0:W]
    xx, yy = xx.ravel(), yy.ravel()
    for _ in range(M):
        jx, jy = rng.random(W * H), rng.random(W * H)
        rr, th = dof.lens_radius * np.sqrt(rng.random(W * H)), 2 * np.pi * rng.random(W * H)
        q = (dof.L.astype(np.float64)[None] + ((xx + jx) / W)[:, None] * dof.U.astype(np.float64)[None]
             + ((yy + jy) / H)[:, None] * dof.V.astype(np.float64)[None])
        o = E[None] + (rr * np.cos(th))[:, None] * u[None] + (rr * np.sin(th))[:, None] * v[None]
        d = E[None] + dof.focus_dist * q - o
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        b = (o * d).sum(1)
        disc = b * b - ((o * o).sum(1) - R * R)
        ref += (disc >= 0) & (-b - np.sqrt(np.maximum(disc, 0)) > 0)
    ref /= M
    nb = 16
    pg, pr = _profile(got, W, H, nb), _profile(ref, W, H, nb)
    assert np.abs(pg - pr).max() < 0.05, (pg.round(3), pr.round(3))
    # soft edge: several partially covered radial bins with DOF, at most one without
    soft = lambda p: ((p > 0.05) & (p < 0.95)).sum()
    assert soft(_profile(got, W, H, nb)) >= 3 and soft(_profile(pin, W, H, nb)) <= 1
    # blur conserves the covered area (disc kernel)
    assert abs(got.sum() - pin.sum()) < 0.03 * pin.sum()
