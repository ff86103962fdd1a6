"""Boundary behaviour on the GPU (include/dpr.h error contract and P:379-431 semantics)."""
import numpy as np
import pytest

import dpr_inputs as di

pytestmark = pytest.mark.gpu


def _dpr():
    from paper_2407_00179_b200 import dpr
    return dpr


def test_state_errors_and_invalid_index():
    dpr = _dpr()
    dev = dpr.Device.create(0, 1, 0)
    try:
        with pytest.raises(dpr.DprError) as e:
            dev.render_frame()                      # before commit_world
        assert e.value.code == -2
        bad = di.Part(0, di.TRIS, verts=di.f32([(0, 0, 0), (1, 0, 0), (0, 1, 0)]),
                      idx=np.array([[0, 1, 7]], np.int32))
        dev.commit_part(bad)
        with pytest.raises(dpr.DprError) as e:
            dev.commit_world()                      # index validated on the GPU
        assert e.value.code == -1 and "index" in str(e.value)
        dev.clear_parts()
        for bad in (di.Part(0, di.SPHERES, spheres=di.f32([[0, 0, 0, 0]])),
                    di.Part(0, di.SPHERES, spheres=di.f32([[0, np.nan, 0, 1]])),
                    di.Part(0, di.TRIS, verts=di.f32([(0, 0, 0), (1, np.inf, 0), (0, 1, 0)]),
                            idx=np.array([[0, 1, 2]], np.int32))):
            dev.commit_part(bad)
            with pytest.raises(dpr.DprError) as e:
                dev.commit_world()                  # finiteness / radius validated on the GPU
            assert e.value.code == -1 and "finite" in str(e.value)
            dev.clear_parts()
        hint = di.Part(0, di.SPHERES, spheres=di.f32([[0, 0, 0, 1]]))
        dev.commit_part(hint)
        dev.commit_world()
        b = dev.get_world_bounds()
        assert np.allclose(b, [-1, -1, -1, 1, 1, 1])
    finally:
        dev.release()


def test_consistency_error_on_every_rank():
    """Frame/Camera must be parameterised identically on all ranks; the
    collective render reports DPR_ERR_CONSISTENCY."""
    dpr = _dpr()
    sc = di.config1()
    devs = dpr.loopback_group(2, 0)
    try:
        for d in devs:
            d.commit_scene_parts(sc.parts)
            d.commit_world()
            d.set_camera(sc.camera)
        devs[0].set_frame(sc.frame)
        devs[1].set_frame(di.Frame(**{**sc.frame.__dict__, "spp": 2}))
        with pytest.raises(dpr.DprError) as e:
            dpr.render_frame_group(devs)
        assert e.value.code == -5
        devs[1].set_frame(sc.frame)
        dpr.render_frame_group(devs)
        assert devs[0].map_frame() is not None
        assert devs[1].map_frame() is None      # undefined on rank != 0, not an error
        assert devs[1].frame_ready()
        st = devs[1].get_stats()
        assert st["nranks"] == 2 and st["S"].shape == (3, 2, 2)
    finally:
        for d in devs:
            d.release()


def test_device_memory_parts_and_rebuild():
    """Parts committed from DEVICE memory (torch tensors) render identically to host parts;
    commit_world can be repeated (the bench step) with identical results."""
    import torch
    dpr = _dpr()
    sc = di.config2(nranks=1, G=31, W=64, H=64, spp=2, spp_batch=2)
    p = sc.parts[0]
    imgs = []
    for device_arrays in (False, True):
        dev = dpr.Device.create(0, 1, 0)
        try:
            if device_arrays:
                q = di.Part(**p.__dict__)
                q.verts = torch.from_numpy(p.verts).cuda()
                q.idx = torch.from_numpy(p.idx).cuda()
                dev.commit_part(q, device_arrays=True)
            else:
                dev.commit_part(p)
            dev.set_camera(sc.camera)
            dev.set_frame(sc.frame)
            for _ in range(2):
                dev.commit_world()
                dev.render_frame()
                imgs.append(dev.map_frame().cpu().numpy().copy())
        finally:
            dev.release()
    for im in imgs[1:]:
        assert np.allclose(im, imgs[0], atol=1e-6)


def test_async_host_commit_and_buffer_recycling():
    """DPR_MEMORY_HOST_ASYNC: pinned host geometry uploaded on the side copy stream while the
    previous frame is still rendering, recycled geometry buffers across clear/commit cycles
    (different sizes, then the same), then a synchronous commit into recycled buffers: every
    frame equals the synchronous-commit render of the same world, bit for bit."""
    import torch
    dpr = _dpr()
    scA = di.config2(nranks=1, G=41, W=48, H=40, spp=2, spp_batch=2)
    scB = di.config2(nranks=1, G=33, W=48, H=40, spp=2, spp_batch=2)

    def pinned(parts):
        out = []
        for p in parts:
            q = di.Part(**p.__dict__)
            if p.kind == di.TRIS:
                q.verts = torch.from_numpy(np.ascontiguousarray(p.verts)).pin_memory().numpy()
                q.idx = torch.from_numpy(np.ascontiguousarray(p.idx)).pin_memory().numpy()
            out.append(q)
        return out

    fr = di.Frame(**{**scA.frame.__dict__, "flags": scA.frame.flags | dpr.DPR_FLAG_DEBUG_DUMPS})

    def render(dev, parts, mode):
        dev.clear_parts()
        for p in parts:
            dev.commit_part(p, async_copy=(mode == "async"))
        dev.commit_world()
        dev.set_camera(scA.camera)
        dev.set_frame(fr)
        dev.render_frame()
        e, o = dev.get_debug(fr.spp, fr.max_depth, fr.W * fr.H)
        return dev.map_frame().cpu().numpy().copy(), e.cpu().numpy().copy(), o.cpu().numpy().copy()

    def same(a, b):
        # events / occlusion bits are deterministic; pixels only up to float-atomic order
        return np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and np.allclose(a[0], b[0], atol=1e-5)

    ref = {}
    dev = dpr.Device.create(0, 1, 0)
    try:
        ref["A"] = render(dev, scA.parts, "sync")
        ref["B"] = render(dev, scB.parts, "sync")
    finally:
        dev.release()
    dev = dpr.Device.create(0, 1, 0)
    try:
        pa, pb = pinned(scA.parts), pinned(scB.parts)
        for name, parts in [("A", pa), ("B", pb), ("B", pb), ("A", pa), ("A", pa)]:
            assert same(render(dev, parts, "async"), ref[name]), name
        assert same(render(dev, scB.parts, "sync"), ref["B"])
        assert not same(ref["A"], ref["B"])
    finally:
        dev.release()


def test_committed_world_renders_while_next_parts_are_committed():
    """The world of the last commit_world stays renderable (bricks included) while the parts
    of the next world are cleared and committed; commit_world then switches worlds."""
    dpr = _dpr()
    G = 25
    h = float(np.float32(2.0 / (G - 1)))
    tf = di.default_tf(alpha_max=0.4, s0=0.2)
    volA = di.Part(0, di.BRICK, gdims=(G,) * 3, origin=(-1, -1, -1), spacing=(h,) * 3,
                   cell_lo=(0, 0, 0), cell_hi=(G - 1,) * 3, voxels=di.volume_field(G), tf=tf)
    sphB = di.Part(0, di.SPHERES, albedo=(0.9, 0.2, 0.2), spheres=di.f32([[0, 0, 0, 0.7]]))
    W = H = 24
    cam = di.camera_basis((0.3, 1.5, -3.0), (0, -0.2, 0), (0, 1, 0), 50.0, W, H)
    fr = di.Frame(W=W, H=H, spp=2, spp_batch=2, max_depth=2, ao_k=1, ao_radius=0.3, dt=h,
                  light_dir=di.f32(di.normalize((0.2, 1, 0.1))), E=(1, 1, 1), A=(0.2, 0.2, 0.2),
                  flags=dpr.DPR_FLAG_DEBUG_DUMPS)
    dev = dpr.Device.create(0, 1, 0)
    try:
        dev.set_camera(cam)
        dev.set_frame(fr)

        def frame():
            dev.render_frame()
            e, o = dev.get_debug(fr.spp, fr.max_depth, W * H)
            return e.cpu().numpy().copy()

        dev.commit_part(volA)
        dev.commit_world()
        evA = frame()
        assert ((evA & 0x80000000) != 0).any()
        dev.clear_parts()
        dev.commit_part(sphB)
        assert np.array_equal(frame(), evA)          # still world A (its bricks kept alive)
        dev.commit_world()
        evB = frame()
        assert not ((evB & 0x80000000) != 0).any() and (evB[:, 0] >= 2).any()
    finally:
        dev.release()


@pytest.mark.parametrize("nranks", [1, 2, 3, 8, 16])
def test_step_barrier_protocol(nranks):
    """The mailbox step barrier of the device-driven loop (seq-parity double buffering, release
    / acquire over peer memory, error OR-ing), all ranks as blocks of ONE cooperative kernel
    with skewed arrivals: every boundary's gathered sums are right."""
    dpr = _dpr()
    assert dpr.test_step_barrier(0, nranks, 2000) == 0


@pytest.mark.parametrize("n", [1, 7, 4095, 4096, 4097, 3 * 4096 + 17, (1 << 20) + 333])
@pytest.mark.parametrize("dist", ["uniform30", "few", "high_digit", "equal"])
def test_radix_sort_stable(n, dist):
    """The LBVH builder's key sort (north star subsystem (1)): ascending keys, equal keys in
    input order -- the stable argsort -- over ragged tile counts and duplicate-heavy keys."""
    import torch
    dpr = _dpr()
    rng = np.random.default_rng(n + len(dist))
    if dist == "uniform30":
        k = rng.integers(0, 1 << 30, n, dtype=np.uint32)
    elif dist == "few":
        k = rng.integers(0, 16, n, dtype=np.uint32) * np.uint32(0x01010101)
    elif dist == "high_digit":
        k = (rng.integers(0, 64, n, dtype=np.uint32) << np.uint32(24)) | np.uint32(5)
    else:
        k = np.full(n, 0x2aaaaaaa, np.uint32)
    kd = torch.from_numpy(k.view(np.int32)).cuda()
    pd = torch.empty(n, dtype=torch.int32, device="cuda")
    dpr.test_radix_sort(0, kd.data_ptr(), n, pd.data_ptr())
    perm = pd.cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(perm, np.argsort(k, kind="stable").astype(np.uint32))
    assert np.array_equal(kd.cpu().numpy().view(np.uint32), k)   # keys untouched


def test_radix_sort_args():
    dpr = _dpr()
    dpr.test_radix_sort(0, 0, 0, 0)                  # n = 0: nothing to do
    with pytest.raises(dpr.DprError):
        dpr.test_radix_sort(0, 0, 5, 0)


def test_brick_row_limit():
    """dpr.h BRICK: a brick stores fewer than 2^31 voxel rows (y * z extent); larger ones are
    rejected at commit_part, before the voxel array is read (the march indexes rows in 32 bits)."""
    dpr = _dpr()
    G = 70000
    tf = di.default_tf()
    big = di.Part(0, di.BRICK, gdims=(4, G, G), origin=(0, 0, 0), spacing=(1e-3,) * 3,
                  cell_lo=(0, 0, 0), cell_hi=(3, 46341, 46341), voxels=np.zeros(8, np.float32), tf=tf)
    dev = dpr.Device.create(0, 1, 0)
    try:
        with pytest.raises(dpr.DprError) as e:
            dev.commit_part(big)
        assert e.value.code == -1 and "rows" in str(e.value)
    finally:
        dev.release()
