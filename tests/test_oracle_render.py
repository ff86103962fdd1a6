"""Oracle pins, part 2: whole-frame behaviour checked against closed forms, hand-derived
routing cases and the paper's invariant (a data-parallel render equals a single-rank render
of the union; P:657-659 S5.2, P:1102-1109 S7.1)."""
import json
import math
import os

import numpy as np
import pytest

import dpr_inputs as di
import oracle as orc


def _plane_scene(extent=50.0, albedo=(0.7, 0.5, 0.3), y=0.0):
    v, i = di.quad_tris([(-extent, y, -extent), (extent, y, -extent), (extent, y, extent),
                         (-extent, y, extent)])
    return di.Part(0, di.TRIS, albedo=albedo, verts=v, idx=i)


def _render(parts, nranks, cam, fr, dp=False, pixels=None):
    return orc.render(orc.OracleScene(parts, nranks), cam, fr, pixels=pixels, dp=dp)


def test_unoccluded_plane_closed_form():
    """P6 closed form (1): on an unoccluded plane every AO ray escapes, so the pixel is
    rho*(E*max(0,n.l) + A) with no Monte Carlo noise; the bounce escapes and adds 0."""
    rho = np.array([0.7, 0.5, 0.3])
    l = di.normalize((0.3, 1.0, 0.2))
    W = H = 16
    cam = di.camera_basis((0, 3, -3), (0, 0, 0), (0, 1, 0), 30.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=1, max_depth=2, ao_k=4, ao_radius=np.inf,
                  light_dir=di.f32(l), E=(1.0, 0.9, 0.8), A=(0.3, 0.3, 0.3), B=(1, 0, 1))
    r = _render([_plane_scene(albedo=rho)], 1, cam, fr)
    cosl = float(np.float32(l[1]))
    exp = rho * (np.array([1.0, 0.9, 0.8]) * cosl + 0.3)
    assert np.allclose(r.rgba[:, :3], exp, atol=2e-6)
    assert (r.rgba[:, 3] == 1.0).all()
    # every AO/shadow bit set (all unoccluded), events are surface hits of id 0/1
    assert (r.occl[:, 0] == 0b11111).all() and (r.occl[:, 1] == 0).all()
    assert set(np.unique(r.events[:, 0])) <= {2, 3}
    assert (r.events[:, 1] == 1).all()  # the bounce escapes to the sky (miss)


def test_sphere_alone_closed_form():
    """P6 closed form (2): a convex sphere never occludes its own AO rays -> AO = 1, pixel =
    rho*(E*max(0,n.l)+A) with n the analytic normal; misses give B, coverage 0."""
    W = H = 24
    cam = di.camera_basis((0, 0, -4), (0, 0, 0), (0, 1, 0), 40.0, W, H)
    l = di.f32(di.normalize((1, 1, -1)))
    fr = di.Frame(W=W, H=H, spp=1, max_depth=1, ao_k=3, light_dir=l, E=(1, 1, 1),
                  A=(0.25, 0.25, 0.25), B=(0.1, 0.2, 0.3), flags=1)
    rho = np.array([0.9, 0.6, 0.3])
    part = di.Part(0, di.SPHERES, albedo=rho, spheres=di.f32([[0, 0, 0, 1]]))
    r = _render([part], 1, cam, fr)
    hits = r.rgba[:, 3] == 1
    assert 100 < hits.sum() < W * H
    assert np.allclose(r.rgba[~hits, :3], [0.1, 0.2, 0.3], atol=1e-7)
    for p in np.nonzero(hits)[0][::7]:
        o, d = orc.camera_ray(cam, fr, int(p))
        o, d = o.astype(np.float64), d.astype(np.float64)
        b = o @ d
        t = -b - math.sqrt(b * b - (o @ o - 1))
        n = o + t * d
        exp = rho * (max(0.0, n @ l.astype(np.float64)) + 0.25)
        assert np.allclose(r.rgba[p, :3], exp, atol=1e-5), (p, r.rgba[p], exp)


def test_empty_world_and_dark_lights():
    """P6 closed forms (3)+(4): an empty world gives B everywhere with coverage 0; E=A=0
    gives 0 except the background."""
    W = H = 8
    cam = di.camera_basis((0, 0, -4), (0, 0, 0), (0, 1, 0), 40.0, W, H)
    fr = di.Frame(W=W, H=H, spp=3, max_depth=2, ao_k=2, B=(0.2, 0.4, 0.6))
    r = _render([], 1, cam, fr)
    assert np.allclose(r.rgba, [0.2, 0.4, 0.6, 0.0], atol=1e-7)
    assert (r.events[:, 0] == 1).all() and (r.events[:, 1] == 0).all()
    part = di.Part(0, di.SPHERES, albedo=(1, 1, 1), spheres=di.f32([[0, 0, 0, 1]]))
    fr0 = di.Frame(W=W, H=H, spp=2, max_depth=2, ao_k=2, E=(0, 0, 0), A=(0, 0, 0), B=(0.2, 0.4, 0.6))
    r = _render([part], 1, cam, fr0)
    cov = r.rgba[:, 3]
    assert np.allclose(r.rgba[:, :3], (1 - cov)[:, None] * np.array([0.2, 0.4, 0.6]), atol=1e-7)


def test_ao_sphere_form_factor():
    """P6 closed form (5): cosine-weighted AO under a sphere of radius R whose centre is at
    distance d and angle theta from the normal (fully above the horizon) is
    1 - (R/d)^2 cos(theta).  E=0, A=1, rho=1 -> pixel = AO fraction."""
    R, c = 0.5, np.array([1.5, 1.5, 0.0])
    d = np.linalg.norm(c)
    expected = 1 - (R / d) ** 2 * (c[1] / d)
    cam = di.camera_basis((-3, 3, 0.0), (0, 0, 0), (0, 1, 0), 1.0, 1, 1)
    K, spp = 16, 2048
    fr = di.Frame(W=1, H=1, spp=spp, spp_batch=spp, max_depth=1, ao_k=K, ao_radius=np.inf,
                  E=(0, 0, 0), A=(1, 1, 1), flags=1)
    parts = [_plane_scene(albedo=(1, 1, 1)),
             di.Part(0, di.SPHERES, albedo=(1, 1, 1), spheres=di.f32([[*c, R]]))]
    r = _render(parts, 1, cam, fr)
    sigma = math.sqrt(expected * (1 - expected) / (K * spp))
    assert abs(r.rgba[0, 0] - expected) < 4 * sigma, (r.rgba[0, 0], expected, sigma)
    # AO radius shorter than the gap to the sphere -> nothing occludes
    fr2 = di.Frame(W=1, H=1, spp=64, max_depth=1, ao_k=K, ao_radius=0.5, E=(0, 0, 0),
                   A=(1, 1, 1), flags=1)
    assert abs(_render(parts, 1, cam, fr2).rgba[0, 0] - 1.0) < 1e-6


def test_shadow_ray_blocked():
    """P6: a point whose light direction is blocked by a sphere gets only ambient."""
    cam = di.camera_basis((-3, 3, 0.0), (0, 0, 0), (0, 1, 0), 1.0, 1, 1)
    fr = di.Frame(W=1, H=1, spp=1, max_depth=1, ao_k=0, light_dir=(0, 1, 0), E=(1, 1, 1),
                  A=(0, 0, 0), flags=1)
    parts = [_plane_scene(albedo=(0.5, 0.5, 0.5)),
             di.Part(0, di.SPHERES, albedo=(1, 1, 1), spheres=di.f32([[0, 2, 0, 0.5]]))]
    r = _render(parts, 1, cam, fr)
    assert r.rgba[0, 0] == 0.0 and r.occl[0, 0, 0] == 0
    r = _render(parts[:1], 1, cam, fr)
    assert abs(r.rgba[0, 0] - 0.5) < 1e-7 and r.occl[0, 0, 0] == 1


@pytest.mark.parametrize("case", ["H1", "H2", "H3", "H4", "H5"])
def test_routing_hand_cases(case, golden_dir):
    """P8 routing + P8b steps, hand-derived (tests/golden/routing_hand_cases.json); H4 is
    the equal-t0 rank tie of the visit key (t0_r, r)."""
    g = json.load(open(os.path.join(golden_dir, "routing_hand_cases.json")))[case]
    sc = di.routing_hand_case(case)
    r = _render(sc.parts, 2, sc.camera, sc.frame, dp=True)
    assert r.S[0].tolist() == g["S_path"]
    assert r.S[1].tolist() == g["S_shadow"]
    assert r.S[2].tolist() == g["S_ao"]
    assert r.V[0].tolist() == g["V_path"] and r.V[1].tolist() == g["V_shadow"]
    assert int(r.events[0, 0, 0]) == g["event"]
    assert int(r.occl[0, 0, 0]) == g["occl"]
    assert np.allclose(r.rgba[0], g["rgba"], atol=1e-7)
    assert r.steps.tolist() == [g["steps"]]
    # per-step matrices (P8b): entries of each step, hand-derived
    rs = orc.render(orc.OracleScene(sc.parts, 2), sc.camera, sc.frame, dp=True, step_matrices=True)
    assert len(rs.S_step) == g["steps"]
    for k in range(g["steps"]):
        assert sorted(np.argwhere(rs.S_step[k]).tolist()) == sorted(g["S_steps"][k]), k
        assert (rs.S_step[k][rs.S_step[k] != 0] == 1).all()
        assert sorted(np.argwhere(rs.V_step[k]).tolist()) == sorted(g["V_steps"][k]), k
    u = _render(di.union_parts(sc.parts), 1, sc.camera, sc.frame)
    assert np.array_equal(u.events, r.events) and np.allclose(u.rgba, r.rgba, atol=1e-12)


def _assert_same_image(a, b):
    assert np.array_equal(a.events, b.events)
    assert np.array_equal(a.occl, b.occl)
    assert np.array_equal(a.gen, b.gen)
    assert np.allclose(a.rgba, b.rgba, atol=1e-12, rtol=0)


def test_config1_dp_equals_union():
    """The paper's invariant on configs[0]: the 2-rank data-parallel render (ray forwarding,
    routing simulator) equals the 1-rank render of the union -- events, occlusion bits and
    pixels -- and has cross-rank shadows (S_shadow != 0) that compositing cannot produce
    (P:645-647)."""
    sc = di.config1()
    r = _render(sc.parts, 2, sc.camera, sc.frame, dp=True)
    u = _render(di.union_parts(sc.parts), 1, sc.camera, sc.frame)
    _assert_same_image(r, u)
    assert r.S[1, 0, 1] + r.S[1, 1, 0] > 0 and r.S[0, 0, 1] + r.S[0, 1, 0] > 0
    # conservation: every forward is one more visit (P8)
    for k in range(3):
        assert r.V[k].sum() >= r.S[k].sum()
    assert r.gen[0] == 64 * 64 + (r.events[:, 1] != 0).sum()


def test_single_rank_has_no_routing():
    """P:1102-1109 (S7.1): a single rank is a plain renderer: S == 0; depth-2 frame takes
    3 steps (primary, then shadow/AO + bounce, then the bounce's shadow/AO)."""
    sc = di.config1()
    u = _render(di.union_parts(sc.parts), 1, sc.camera, sc.frame, dp=True)
    assert (u.S == 0).all()
    assert u.steps.tolist() == [3]
    # one rank: each ray is traced at most once (no-candidate rays are never traced)
    assert (u.V[:, 0] <= u.gen).all() and u.V[0, 0] > 0.9 * 4096


def _random_world(seed, ntri=120, nsph=40):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1, 1, size=(ntri, 1, 3))
    v = (c + rng.uniform(-0.25, 0.25, size=(ntri, 3, 3))).astype(np.float32).reshape(-1, 3)
    sp = np.concatenate([rng.uniform(-1, 1, (nsph, 3)), rng.uniform(0.05, 0.2, (nsph, 1))], 1)
    return v, sp.astype(np.float32)


@pytest.mark.parametrize("nranks,seed", [(2, 0), (3, 1), (4, 2), (8, 3)])
def test_partition_independence(nranks, seed):
    """A random prim->rank reassignment (not spatial: boxes overlap heavily) leaves events,
    occlusion bits and pixels unchanged (SURVEY 8(c).4 partition independence)."""
    v, sp = _random_world(seed)
    rng = np.random.default_rng(100 + seed)
    tri_rank = rng.integers(0, nranks, size=v.shape[0] // 3)
    sph_rank = rng.integers(0, nranks, size=sp.shape[0])
    parts = []
    for r in range(nranks):
        tv = v.reshape(-1, 3, 3)[tri_rank == r].reshape(-1, 3)
        if tv.shape[0]:
            parts.append(di.Part(r, di.TRIS, albedo=(0.6 + 0.05 * r, 0.5, 0.4), verts=tv,
                                 idx=np.arange(tv.shape[0], dtype=np.int32).reshape(-1, 3)))
        s = sp[sph_rank == r]
        if s.shape[0]:
            parts.append(di.Part(r, di.SPHERES, albedo=(0.3, 0.7, 0.2 + 0.05 * r), spheres=s))
    W = H = 24
    cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=1, max_depth=3, ao_k=2, ao_radius=0.6,
                  light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1),
                  A=(0.3, 0.3, 0.3), B=(0.1, 0.1, 0.2))
    dpres = _render(parts, nranks, cam, fr, dp=True)
    u = _render(di.union_parts(parts), 1, cam, fr)
    # ids differ between the partitioned and the union world only by the permutation the
    # concatenation order induces; both are the same list here (union_parts keeps rank order)
    _assert_same_image(dpres, u)
    assert dpres.S.sum() > 0
    assert len(dpres.steps) == 2
    # P8b per-step matrices add up to the frame totals; a step's visits at rank r are the rays
    # queued for r by the previous step (forwards + spawns into r, or kept primaries at step 0)
    st = orc.render(orc.OracleScene(parts, nranks), cam, fr, dp=True, step_matrices=True)
    assert np.array_equal(st.S_step.sum(axis=0), dpres.S) and np.array_equal(st.V_step.sum(axis=0), dpres.V)
    assert len(st.S_step) == dpres.steps.sum()


def _const_volume(G, value, alpha, nbricks=1, nranks=1):
    tf = np.zeros((256, 4), np.float32)
    tf[:, :3] = (0.2, 0.5, 0.8)
    tf[:, 3] = alpha
    h = np.float32(2.0 / (G - 1))
    parts = []
    for r, (lo, hi) in enumerate(di.brick_boxes((G - 1,) * 3, nbricks)):
        nx, ny, nz = hi[0] - lo[0] + 1, hi[1] - lo[1] + 1, hi[2] - lo[2] + 1
        parts.append(di.Part(r % nranks, di.BRICK, gdims=(G,) * 3, origin=(-1, -1, -1),
                             spacing=(float(h),) * 3, cell_lo=lo, cell_hi=hi,
                             voxels=np.full((nz, ny, nx), value, np.float32), tf=tf))
    return parts, float(h)


def test_volume_first_collision_is_geometric():
    """P10: with a constant alpha field the index of the first colliding sample is
    geometric: P(j) = (1-alpha)^j alpha (j counted from the first sample inside).  Pins the
    per-sample Philox draws (purpose 4) and the collision rule u_i < alpha_i."""
    alpha = 0.1
    parts, h = _const_volume(17, 0.5, alpha)
    cam = di.camera_basis((0.05, 0.03, -3), (0.05, 0.03, 0), (0, 1, 0), 1.0, 1, 1)
    spp = 6000
    fr = di.Frame(W=1, H=1, spp=spp, spp_batch=spp, max_depth=1, ao_k=0, dt=h, E=(0, 0, 0),
                  flags=1)
    r = _render(parts, 1, cam, fr)
    ev = r.events[:, 0, 0]
    vol = ev[(ev & 0x80000000) != 0] & 0x7FFFFFFF
    i0 = vol.min()
    j = vol - i0
    n_inside = 16  # samples inside the 2-wide box at dt = 2/16
    pm = (1 - alpha) ** np.arange(n_inside + 2) * alpha
    p_any = 1 - (1 - alpha) ** n_inside
    assert abs(len(vol) / spp - p_any) < 4 * math.sqrt(p_any * (1 - p_any) / spp)
    for k in range(4):
        pk = pm[k]
        assert abs((j == k).mean() * len(vol) / spp - pk) < 4 * math.sqrt(pk * (1 - pk) / spp)
    # coverage counts volume events; rgb = 0 because E=0
    assert abs(r.rgba[0, 3] - len(vol) / spp) < 1e-12


def test_volume_transmittance_of_shadow_rays():
    """P10 binary shadows: the fraction of unoccluded shadow rays through a constant-alpha
    slab of n samples is (1-alpha)^n in expectation (Beer-Lambert on the sample grid)."""
    alpha, G = 0.05, 9
    parts, h = _const_volume(G, 0.5, alpha)
    plane = _plane_scene(extent=3, albedo=(1, 1, 1), y=-1.5)
    cam = di.camera_basis((0.01, -1.0, -3.0), (0.01, -1.5, 0.0), (0, 1, 0), 1.0, 1, 1)
    spp = 3000
    fr = di.Frame(W=1, H=1, spp=spp, spp_batch=spp, max_depth=1, ao_k=0, dt=h,
                  light_dir=(0, 1, 0), E=(1, 1, 1), flags=1)
    r = _render(parts + [plane], 1, cam, fr)
    # the shadow ray from the plane goes straight up through 8 cells = 8 samples
    p = (1 - alpha) ** 8
    assert abs(r.rgba[0, 0] - p) < 4 * math.sqrt(p * (1 - p) / spp)


@pytest.mark.parametrize("nbricks,nranks", [(2, 1), (4, 1), (4, 4), (8, 2), (3, 3)])
def test_brick_split_equals_single_grid(nbricks, nranks):
    """P10: splitting the grid into bricks (on one rank or across ranks)
    reproduces the single-grid render bit-exactly: global-coordinate sampling + half-open
    ownership.  Also the routing simulator (dp) equals the union renderer."""
    G = 17
    field = di.volume_field(G)
    tf = di.default_tf(alpha_max=0.6, s0=0.2)

    def bricks(nb, nr):
        h = np.float32(2.0 / (G - 1))
        out = []
        for r, (lo, hi) in enumerate(di.brick_boxes((G - 1,) * 3, nb)):
            vox = field[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
            out.append(di.Part(r % nr, di.BRICK, gdims=(G,) * 3, origin=(-1, -1, -1),
                               spacing=(float(h),) * 3, cell_lo=lo, cell_hi=hi,
                               voxels=np.ascontiguousarray(vox), tf=tf))
        return out, float(h)

    single, h = bricks(1, 1)
    split, _ = bricks(nbricks, nranks)
    W = H = 20
    cam = di.camera_basis((0.4, 0.7, 2.6), (0, 0, 0), (0, 1, 0), 40.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=1, max_depth=2, ao_k=0, dt=h,
                  light_dir=di.f32(di.normalize((1, 2, 1))), E=(1, 1, 1))
    a = _render(single, 1, cam, fr)
    b = _render(split, nranks, cam, fr, dp=True)
    c = _render(di.union_parts(split), 1, cam, fr)
    assert ((a.events & 0x80000000) != 0).sum() > 50
    _assert_same_image(a, b)
    _assert_same_image(a, c)


def test_mixed_surface_volume_tie_rules():
    """P9: volume ids 0x80000000|i compare above every surface id, so a surface wins a tie;
    mixed world dp == union."""
    G = 9
    parts, h = _const_volume(G, 0.5, 0.3, nbricks=2, nranks=2)
    sph = di.Part(1, di.SPHERES, albedo=(0.9, 0.1, 0.1), spheres=di.f32([[0.2, 0.1, 0.0, 0.4]]))
    pl = _plane_scene(extent=3, albedo=(0.5, 0.5, 0.5), y=-1.2)
    pl.rank = 0
    allp = parts + [sph, pl]
    W = H = 16
    cam = di.camera_basis((0.3, 1.5, -3.0), (0, -0.5, 0), (0, 1, 0), 50.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=2, max_depth=2, ao_k=1, ao_radius=0.3, dt=h,
                  light_dir=di.f32(di.normalize((0.2, 1, 0.1))), E=(1, 1, 1), A=(0.2, 0.2, 0.2))
    r = _render(allp, 2, cam, fr, dp=True)
    u = _render(di.union_parts(allp), 1, cam, fr)
    _assert_same_image(r, u)
    ev = r.events[:, 0]
    assert ((ev & 0x80000000) != 0).any() and ((ev >= 2) & (ev < 0x80000000)).any()


def test_deep_composite_over_operator():
    """deepComp's over operator (SPEC S:452 worked example): a half-transparent
    red fragment in front of an opaque blue one -> (0.5, 0, 0.5, 1); depth order, not rank
    order, decides; the background fills what is left."""
    red = [0.5, 0.0, 0.0, 0.5]   # premultiplied, alpha 0.5
    blue = [0.0, 0.0, 1.0, 1.0]
    rgba = np.array([[blue], [red]], np.float64)          # rank 0 blue, rank 1 red
    depth = np.array([[2.0], [1.0]], np.float32)          # red is in front
    out = orc.deep_composite(rgba, depth, (0.1, 0.2, 0.3))
    assert np.allclose(out[0], [0.5, 0.0, 0.5, 1.0])
    out = orc.deep_composite(rgba[:1] * 0, np.array([[np.inf]], np.float32), (0.1, 0.2, 0.3))
    assert np.allclose(out[0], [0.1, 0.2, 0.3, 0.0])
    # equal depth: lower rank first
    two = np.array([[[0.2, 0, 0, 0.5]], [[0, 0.2, 0, 0.5]]])
    out = orc.deep_composite(two, np.array([[1.0], [1.0]], np.float32), (0, 0, 0))
    assert np.allclose(out[0], [0.2, 0.1, 0, 0.75])


def test_local_fragments_union_invariance():
    """One rank holding the whole boxes scene: local fragments composited == the plain
    render (compositing is the identity for N=1)."""
    sc = di.boxes_scene(nranks=1, W=24, H=24, spp=2)
    rgba, depth = orc.render_local_fragments(sc.parts, 0, sc.camera, sc.frame)
    comp = orc.deep_composite(rgba[None], depth[None], sc.frame.B)
    u = orc.render(orc.OracleScene(sc.parts, 1), sc.camera, sc.frame)
    assert np.allclose(comp, u.rgba, atol=1e-9)
