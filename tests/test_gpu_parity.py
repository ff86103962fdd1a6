"""CUDA path (libdpr.so through the C ABI) vs the oracle, element by element on the same
seeded inputs.  Bit-exact: hit/event codes, occlusion bits, rays generated, routing
matrices S, visits V, step counts.  Pixels: max-abs 1e-3 / mean-abs 1e-4 per channel
(north_star).  N>1 runs the SAME kernels as N virtual ranks on one GPU (loopback group)."""
import numpy as np
import pytest

import dpr_inputs as di
from tests.gpu_helpers import assert_parity, gpu_render, oracle_render

pytestmark = pytest.mark.gpu


def test_config1_single_rank_union():
    """configs[0] union world on one rank (one rank == plain renderer)."""
    sc = di.config1()
    parts = di.union_parts(sc.parts)
    g = gpu_render(parts, 1, sc.camera, sc.frame)
    o = oracle_render(parts, 1, sc.camera, sc.frame)
    assert_parity(g, o)


def test_config1_two_ranks():
    """configs[0] as specified: two ranks split by x-half, ray forwarding with cross-rank
    shadows; routing matrices bit-exact against the oracle's routing simulator."""
    sc = di.config1()
    g = gpu_render(sc.parts, 2, sc.camera, sc.frame)
    o = oracle_render(sc.parts, 2, sc.camera, sc.frame)
    assert_parity(g, o)
    assert o.S[1].sum() > 0


@pytest.mark.parametrize("case", ["H1", "H2", "H3", "H4", "H5"])
def test_routing_hand_cases(case):
    sc = di.routing_hand_case(case)
    g = gpu_render(sc.parts, 2, sc.camera, sc.frame)
    o = oracle_render(sc.parts, 2, sc.camera, sc.frame)
    assert_parity(g, o)


def _random_world(seed, nranks, ntri=300, nsph=80):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1, 1, size=(ntri, 1, 3))
    v = (c + rng.uniform(-0.25, 0.25, size=(ntri, 3, 3))).astype(np.float32)
    sp = np.concatenate([rng.uniform(-1, 1, (nsph, 3)), rng.uniform(0.05, 0.2, (nsph, 1))], 1).astype(np.float32)
    tr = rng.integers(0, nranks, ntri)
    srk = rng.integers(0, nranks, nsph)
    parts = []
    for r in range(nranks):
        tv = v[tr == r].reshape(-1, 3)
        if tv.shape[0]:
            parts.append(di.Part(r, di.TRIS, albedo=(0.6, 0.5 + 0.03 * r, 0.4), verts=tv,
                                 idx=np.arange(tv.shape[0], dtype=np.int32).reshape(-1, 3)))
        s = sp[srk == r]
        if s.shape[0]:
            parts.append(di.Part(r, di.SPHERES, albedo=(0.3, 0.7, 0.2), spheres=s))
    return parts


@pytest.mark.parametrize("nranks,seed", [(1, 0), (2, 1), (3, 2), (4, 3), (8, 4)])
def test_random_world_partitions(nranks, seed):
    """Overlapping random partitions (not spatial), depth 3, AO + shadows + bounces."""
    parts = _random_world(seed, nranks)
    W = H = 48
    cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    fr = di.Frame(W=W, H=H, spp=3, spp_batch=2, max_depth=3, ao_k=2, ao_radius=0.6,
                  light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3),
                  B=(0.1, 0.1, 0.2))
    g = gpu_render(parts, nranks, cam, fr)
    o = oracle_render(parts, nranks, cam, fr)
    assert_parity(g, o)


def _volume_scene(G, nbricks, nranks, alpha_max=0.6):
    field = di.volume_field(G)
    tf = di.default_tf(alpha_max=alpha_max, s0=0.2)
    h = np.float32(2.0 / (G - 1))
    parts = []
    for r, (lo, hi) in enumerate(di.brick_boxes((G - 1,) * 3, nbricks)):
        vox = field[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
        parts.append(di.Part(r % nranks, di.BRICK, gdims=(G,) * 3, origin=(-1, -1, -1),
                             spacing=(float(h),) * 3, cell_lo=lo, cell_hi=hi,
                             voxels=np.ascontiguousarray(vox), tf=tf))
    return parts, float(h)


MARCH_MODES = {"auto": None, "inline": "0", "group1": "1000000000:1", "group4": "1000000000:4",
               "group32": "1000000000:32"}


@pytest.mark.parametrize("march", list(MARCH_MODES))
@pytest.mark.parametrize("nbricks,nranks", [(1, 1), (4, 1), (2, 2), (4, 4), (8, 8)])
def test_volume_bricks(nbricks, nranks, march, monkeypatch):
    """P10 stochastic DVR + binary volume shadows + isotropic bounce, bricks per rank; the
    march inside the trace kernels (one lane per ray) and in k_march_* (G lanes per ray)."""
    if MARCH_MODES[march] is not None:
        monkeypatch.setenv("DPR_MARCH", MARCH_MODES[march])
    parts, h = _volume_scene(41, nbricks, nranks)
    W = H = 40
    cam = di.camera_basis((0.4, 0.7, 2.6), (0, 0, 0), (0, 1, 0), 40.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=2, max_depth=2, dt=h,
                  light_dir=di.f32(di.normalize((1, 2, 1))), E=(1, 1, 1))
    g = gpu_render(parts, nranks, cam, fr)
    o = oracle_render(parts, nranks, cam, fr)
    assert ((o.events & 0x80000000) != 0).sum() > 100
    assert_parity(g, o)


def test_mixed_surfaces_and_volume():
    parts, h = _volume_scene(33, 2, 2, alpha_max=0.3)
    parts.append(di.Part(1, di.SPHERES, albedo=(0.9, 0.1, 0.1), spheres=di.f32([[0.2, 0.1, 0.0, 0.4]])))
    v, i = di.quad_tris([(-3, -1.2, -3), (3, -1.2, -3), (3, -1.2, 3), (-3, -1.2, 3)])
    parts.append(di.Part(0, di.TRIS, albedo=(0.5, 0.5, 0.5), verts=v, idx=i))
    W = H = 32
    cam = di.camera_basis((0.3, 1.5, -3.0), (0, -0.5, 0), (0, 1, 0), 50.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=1, max_depth=2, ao_k=1, ao_radius=0.3, dt=h,
                  light_dir=di.f32(di.normalize((0.2, 1, 0.1))), E=(1, 1, 1), A=(0.2, 0.2, 0.2))
    g = gpu_render(parts, 2, cam, fr)
    o = oracle_render(parts, 2, cam, fr)
    assert_parity(g, o)


def test_occlusion_resolve_fused_and_separate(monkeypatch):
    """One rank: k_trace_occl resolves its rays itself (fused, the default) or k_resolve_occl
    does (DPR_NO_FUSE_RESOLVE=1); both equal the oracle (events, occlusion bits, visits V),
    and the fused frame launches one kernel less per occlusion wavefront."""
    sc = di.config2(nranks=1, G=41, W=96, H=80, spp=4, spp_batch=2)
    o = oracle_render(sc.parts, 1, sc.camera, sc.frame)
    assert_parity(gpu_render(sc.parts, 1, sc.camera, sc.frame), o)  # device-driven loop
    # launch accounting on the host loop (the device loop launches k_resolve_occl always; it
    # exits at once when the trace resolved the queue)
    monkeypatch.setenv("DPR_STEP_LOOP", "host")
    fused = gpu_render(sc.parts, 1, sc.camera, sc.frame)
    assert_parity(fused, o)
    monkeypatch.setenv("DPR_NO_FUSE_RESOLVE", "1")
    sep = gpu_render(sc.parts, 1, sc.camera, sc.frame)
    assert_parity(sep, o)
    n_occl = sep[3]["trace_occl_launches"]
    assert n_occl > 0
    assert sep[3]["kernel_launches_local"] - fused[3]["kernel_launches_local"] == n_occl


@pytest.mark.parametrize("nranks", [1, 4])
def test_config2_family_small(nranks):
    """configs[1] family at a size the oracle finishes in seconds: ~180k-triangle gyroid,
    spatially bisected over N ranks, 96x80 (ragged tiles), 4 spp in 2 batches, shadows +
    AO (K=4, r=0.25, depth 1)."""
    sc = di.config2(nranks=nranks, G=41, W=96, H=80, spp=4, spp_batch=2)
    g = gpu_render(sc.parts, nranks, sc.camera, sc.frame)
    o = oracle_render(sc.parts, nranks, sc.camera, sc.frame)
    assert_parity(g, o)


def test_empty_world_and_empty_rank():
    """Degenerate cases: an empty world (background, coverage 0) and a rank with no parts."""
    W = H = 16
    cam = di.camera_basis((0, 0, -4), (0, 0, 0), (0, 1, 0), 40.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, max_depth=2, ao_k=2, B=(0.2, 0.4, 0.6))
    g = gpu_render([], 1, cam, fr)
    assert np.allclose(g[0], [0.2, 0.4, 0.6, 0.0], atol=1e-6)
    parts = [di.Part(1, di.SPHERES, albedo=(1, 1, 1), spheres=di.f32([[0, 0, 0, 1]]))]
    g = gpu_render(parts, 3, cam, fr)
    o = oracle_render(parts, 3, cam, fr)
    assert_parity(g, o)


def test_single_triangle_and_single_sphere():
    W = H = 16
    cam = di.camera_basis((0, 0, -4), (0, 0, 0), (0, 1, 0), 40.0, W, H)
    fr = di.Frame(W=W, H=H, spp=1, max_depth=2, ao_k=1, light_dir=(0, 0, -1), E=(1, 1, 1), A=(0.2, 0.2, 0.2))
    for part in [di.Part(0, di.TRIS, verts=di.f32([(-1, -1, 0), (1, -1, 0), (0, 1, 0)]),
                         idx=np.array([[0, 1, 2]], np.int32)),
                 di.Part(0, di.SPHERES, spheres=di.f32([[0, 0, 0, 0.7]]))]:
        g = gpu_render([part], 1, cam, fr)
        o = oracle_render([part], 1, cam, fr)
        assert_parity(g, o)


@pytest.mark.parametrize("nranks", [1, 8])
def test_config4_family_small(nranks):
    """configs[3] family: Gaussian sphere clusters (per-cluster albedo parts) + gyroid mesh,
    partitioned over all prims by centroid bisection, path tracing depth 4, K=1 AO."""
    sc = di.config4(nranks=nranks, n_clusters=24, per_cluster=400, G=41, W=72, H=40, spp=2)
    g = gpu_render(sc.parts, nranks, sc.camera, sc.frame)
    o = oracle_render(sc.parts, nranks, sc.camera, sc.frame)
    assert (o.events[:, 3] != 0).sum() > 100  # paths reach depth 4
    assert_parity(g, o)


def test_config5_family_small():
    """configs[4] family: gyroid mesh + volume bricks on 4 ranks, depth 2, K=1, spp batches."""
    sc = di.config5(nranks=4, G_mesh=51, G_vol=49, W=80, H=45, spp=4, spp_batch=2, alpha_max=0.6)
    g = gpu_render(sc.parts, 4, sc.camera, sc.frame)
    o = oracle_render(sc.parts, 4, sc.camera, sc.frame)
    assert ((o.events & 0x80000000) != 0).sum() > 20
    assert_parity(g, o)


@pytest.mark.parametrize("mode", ["fused", "fused-host", "sendrecv"])
@pytest.mark.parametrize("case", ["c1", "random4", "c2x4"])
def test_exchange_modes(mode, case, monkeypatch):
    """Both exchange implementations give bit-identical routing and images: 'fused' (kernels
    append straight into the destination rank's next queue through peer pointers + remote
    tail atomics) with the device-driven step loop (a CUDA graph per batch)
    or the host loop, and 'sendrecv' (counts allgather + grouped send/recv of per-destination
    send queues)."""
    monkeypatch.setenv("DPR_EXCHANGE", mode.split("-")[0])
    monkeypatch.setenv("DPR_STEP_LOOP", "host" if mode.endswith("host") else "device")
    if case == "c1":
        sc = di.config1()
        parts, n, cam, fr = sc.parts, 2, sc.camera, sc.frame
    elif case == "random4":
        parts, n = _random_world(7, 4), 4
        cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, 40, 40)
        fr = di.Frame(W=40, H=40, spp=2, spp_batch=1, max_depth=3, ao_k=2, ao_radius=0.6,
                      light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3))
    else:
        sc = di.config2(nranks=4, G=41, W=64, H=48, spp=4, spp_batch=2)
        parts, n, cam, fr = sc.parts, 4, sc.camera, sc.frame
    g = gpu_render(parts, n, cam, fr)
    o = oracle_render(parts, n, cam, fr)
    assert_parity(g, o)
    st = g[3]
    rec = sum(int(st["S"][0, 0, q]) * 64 + int(st["S"][1:, 0, q].sum()) * 48 for q in range(1, n))
    assert st["exchanged_bytes_local"] == rec


@pytest.mark.parametrize("strategy", ["roundrobin", "binpack"])
def test_partition_strategies(strategy):
    """NEXT f2: the paper's simple distributions render bit-identically."""
    sc = di.config2(nranks=4, G=41, W=64, H=48, spp=2, spp_batch=2, partition=strategy)
    g = gpu_render(sc.parts, 4, sc.camera, sc.frame)
    o = oracle_render(sc.parts, 4, sc.camera, sc.frame)
    assert_parity(g, o)


@pytest.mark.parametrize("nranks", [1, 3])
def test_depth_of_field(nranks):
    """NEXT f4: thin-lens camera (reading R-DOF).  Primary origins vary per sample,
    so the first-candidate rank of each primary differs too: events, occlusion bits and
    routing bit-exact on the config2 family and on configs[0]."""
    import dataclasses
    sc = di.config2(nranks=nranks, G=41, W=72, H=56, spp=4, spp_batch=2)
    cam = dataclasses.replace(sc.camera, lens_radius=0.15, focus_dist=3.2)
    g = gpu_render(sc.parts, nranks, cam, sc.frame)
    o = oracle_render(sc.parts, nranks, cam, sc.frame)
    assert_parity(g, o)
    c1 = di.config1()
    cam1 = dataclasses.replace(c1.camera, lens_radius=0.3, focus_dist=5.0)
    fr1 = di.Frame(**{**c1.frame.__dict__, "spp": 4, "spp_batch": 4})
    g = gpu_render(c1.parts, 2, cam1, fr1)
    o = oracle_render(c1.parts, 2, cam1, fr1)
    assert_parity(g, o)


@pytest.mark.parametrize("nranks,mode", [(1, "sendrecv"), (3, "sendrecv"), (4, "fused"), (8, "sendrecv")])
def test_ring_schedule(nranks, mode, monkeypatch):
    """NEXT f4: ring schedule (reading R-RING, DPR_FLAG_RING): every ray visits every
    rank in ring order.  Events/occlusion bits/pixels equal the visit rule's, and the ring's
    own routing matrices, visit counts and step counts equal the oracle's simulator."""
    monkeypatch.setenv("DPR_EXCHANGE", mode)
    parts = _random_world(nranks + 10, nranks)
    W = H = 40
    cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    fr = di.Frame(W=W, H=H, spp=3, spp_batch=2, max_depth=3, ao_k=2, ao_radius=0.6,
                  light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3),
                  B=(0.1, 0.1, 0.2), flags=8)
    g = gpu_render(parts, nranks, cam, fr)
    o = oracle_render(parts, nranks, cam, fr)
    assert_parity(g, o)
    if nranks > 1:
        assert (o.V == o.gen[:, None]).all()


def test_ring_schedule_volume_and_config2():
    """Ring schedule with bricks (stochastic DVR, binary volume shadows) and on the config2
    family over 4 spatial ranks."""
    parts, h = _volume_scene(33, 4, 4)
    W = H = 32
    cam = di.camera_basis((0.3, 1.5, -3.0), (0, -0.2, 0), (0, 1, 0), 50.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=2, max_depth=2, ao_k=1, ao_radius=0.3, dt=h,
                  light_dir=di.f32(di.normalize((0.2, 1, 0.1))), E=(1, 1, 1), A=(0.2, 0.2, 0.2), flags=8)
    assert_parity(gpu_render(parts, 4, cam, fr), oracle_render(parts, 4, cam, fr))
    sc = di.config2(nranks=4, G=41, W=64, H=48, spp=2, spp_batch=2)
    fr = di.Frame(**{**sc.frame.__dict__, "flags": 8})
    assert_parity(gpu_render(sc.parts, 4, sc.camera, fr), oracle_render(sc.parts, 4, sc.camera, fr))


@pytest.mark.parametrize("nbricks,nranks", [(1, 1), (4, 2), (8, 4), (8, 8)])
def test_delta_tracking(nbricks, nranks):
    """NEXT f4: delta tracking (DPR_FLAG_DELTA; readings R-DELTA, R-LOG): tentative points
    from the global grid domain entry, pinned log, one global majorant allgathered across
    ranks; events (VOL_BIT | tentative index), occlusion bits, routing bit-exact."""
    parts, h = _volume_scene(41, nbricks, nranks, alpha_max=0.3)
    W = H = 40
    cam = di.camera_basis((0.3, 1.5, -3.0), (0, -0.2, 0), (0, 1, 0), 50.0, W, H)
    fr = di.Frame(W=W, H=H, spp=3, spp_batch=2, max_depth=2, ao_k=1, ao_radius=0.3, dt=h,
                  light_dir=di.f32(di.normalize((0.2, 1, 0.1))), E=(1, 1, 1), A=(0.2, 0.2, 0.2), flags=16)
    g = gpu_render(parts, nranks, cam, fr)
    o = oracle_render(parts, nranks, cam, fr)
    assert ((o.events & 0x80000000) != 0).sum() > 100
    assert_parity(g, o)


def test_delta_tracking_mixed_and_ring():
    """Delta tracking with surfaces in front of / inside the volume, and combined with the
    ring schedule."""
    parts, h = _volume_scene(33, 4, 2, alpha_max=0.3)
    parts.append(di.Part(1, di.SPHERES, albedo=(0.9, 0.1, 0.1), spheres=di.f32([[0.2, 0.1, 0.0, 0.4]])))
    v, i = di.quad_tris([(-3, -1.2, -3), (3, -1.2, -3), (3, -1.2, 3), (-3, -1.2, 3)])
    parts.append(di.Part(0, di.TRIS, albedo=(0.5, 0.5, 0.5), verts=v, idx=i))
    W = H = 32
    cam = di.camera_basis((0.3, 1.5, -3.0), (0, -0.5, 0), (0, 1, 0), 50.0, W, H)
    for flags in (16, 16 | 8):
        fr = di.Frame(W=W, H=H, spp=2, spp_batch=1, max_depth=3, ao_k=1, ao_radius=0.3, dt=h,
                      light_dir=di.f32(di.normalize((0.2, 1, 0.1))), E=(1, 1, 1), A=(0.2, 0.2, 0.2),
                      flags=flags)
        assert_parity(gpu_render(parts, 2, cam, fr), oracle_render(parts, 2, cam, fr))


def test_limits_and_ragged_batches():
    """Edge sizes: ao_k = 30 (the maximum: AO slots use bits 1..30 of the occlusion dump),
    deep paths (max_depth 8) inside a closed sphere (every path ray hits), spp not a multiple
    of spp_batch (ragged last batch), image size not a multiple of the 8x4 ray tiles."""
    parts = [di.Part(0, di.SPHERES, albedo=(0.8, 0.7, 0.6), spheres=di.f32([[0, 0, 0, 3.0]])),
             di.Part(1, di.SPHERES, albedo=(0.2, 0.5, 0.9), spheres=di.f32([[0.4, -0.2, 0.8, 0.5]])),
             di.Part(1, di.TRIS, albedo=(0.9, 0.9, 0.2),
                     verts=di.f32([[-1, -1, 1.5], [1, -1, 1.5], [0, 1, 1.5]]), idx=np.array([[0, 1, 2]], np.int32))]
    W, H = 37, 23
    cam = di.camera_basis((0, 0, -1.5), (0, 0, 1), (0, 1, 0), 70.0, W, H)
    fr = di.Frame(W=W, H=H, spp=5, spp_batch=2, max_depth=8, ao_k=30, ao_radius=0.7,
                  light_dir=di.f32(di.normalize((0.3, 1, -0.2))), E=(1, 1, 1), A=(0.3, 0.3, 0.3),
                  B=(0.1, 0.1, 0.2))
    g = gpu_render(parts, 2, cam, fr)
    o = oracle_render(parts, 2, cam, fr)
    assert ((o.events[:, 7] >= 2) & ((o.events[:, 7] & 0x80000000) == 0)).any()  # depth-8 hits
    assert (o.occl >> 30).any()                                                    # AO ray 29 set
    assert_parity(g, o)


def _with_collinear_triangles(parts, nranks, n=40, seed=9):
    """Add exactly-collinear triangles (binary32 cross(e1,e2) == 0; reading R-DEGEN) spread
    through the world: the generators never make them, a user may."""
    rng = np.random.default_rng(seed)
    f = np.float32
    vs = []
    while len(vs) < n:
        v0 = rng.uniform(-1, 1, 3).astype(f)
        e = rng.uniform(-0.4, 0.4, 3).astype(f)
        v1, v2 = (v0 + e).astype(f), (v0 + f(2) * e).astype(f)  # e2 = 2*e1 exactly
        e1, e2 = v1 - v0, v2 - v0
        ng = np.array([e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                       e1[0] * e2[1] - e1[1] * e2[0]], f)
        if not np.any(ng != 0):
            vs.append(np.stack([v0, v1, v2]))
    out = list(parts)
    for r in range(nranks):
        tv = np.concatenate(vs[r::nranks]).astype(f)
        out.append(di.Part(r, di.TRIS, albedo=(0.9, 0.9, 0.9), verts=tv,
                           idx=np.arange(tv.shape[0], dtype=np.int32).reshape(-1, 3)))
    return out


@pytest.mark.parametrize("nranks", [1, 2])
def test_zero_area_triangles(nranks):
    """Reading R-DEGEN on an un-narrowed input: collinear triangles are never hit (no NaN
    normal, ray or pixel), on the GPU exactly as in the oracle."""
    parts = _with_collinear_triangles(_random_world(5, nranks), nranks)
    W = H = 48
    cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=2, max_depth=2, ao_k=2, ao_radius=0.6,
                  light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3))
    g = gpu_render(parts, nranks, cam, fr)
    o = oracle_render(parts, nranks, cam, fr)
    assert np.isfinite(g[0]).all()
    assert_parity(g, o)


@pytest.mark.parametrize("nranks", [2, 3])
def test_skewed_camera_basis(nranks):
    """primary-generation culling (gen_rect) must hold for ANY camera basis -- here
    an off-axis image region (L shifted by 0.3 U + 0.2 V: U, V no longer perpendicular to the
    view axis) and a sheared V.  Routing and events bit-exact at N > 1."""
    parts = _random_world(11, nranks)
    W, H = 40, 32
    cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    L, U, V = (np.asarray(x, np.float64) for x in (cam.L, cam.U, cam.V))
    cam = di.Camera(E=cam.E, L=di.f32(L + 0.3 * U + 0.2 * V), U=cam.U, V=di.f32(V + 0.25 * U))
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=1, max_depth=2, ao_k=1, ao_radius=0.5,
                  light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3))
    g = gpu_render(parts, nranks, cam, fr)
    o = oracle_render(parts, nranks, cam, fr)
    assert_parity(g, o)


@pytest.mark.parametrize("builder", ["ploc", "karras", "agglo"])
@pytest.mark.parametrize("nranks", [1, 3])
def test_bvh_builders(builder, nranks, monkeypatch):
    """Every binary builder that ships in libdpr.so (DPR_BUILDER: agglomerative LBVH, the
    default; Karras 2012 + bottom-up refit; PLOC) gives the same events, occlusion bits and
    routing as the oracle (traversal result = brute force over the rank's prims, P9)."""
    monkeypatch.setenv("DPR_BUILDER", builder)
    parts = _random_world(21, nranks, ntri=400, nsph=120)
    W = H = 40
    cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=2, max_depth=2, ao_k=2, ao_radius=0.6,
                  light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3))
    g = gpu_render(parts, nranks, cam, fr)
    o = oracle_render(parts, nranks, cam, fr)
    assert_parity(g, o)
    sc = di.config2(nranks=nranks, G=41, W=48, H=40, spp=2, spp_batch=2)
    g = gpu_render(sc.parts, nranks, sc.camera, sc.frame)
    o = oracle_render(sc.parts, nranks, sc.camera, sc.frame)
    assert_parity(g, o)
