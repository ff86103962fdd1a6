"""Oracle pins for the ring schedule (P:232 S2.2 "wave-fronts are exchanged in a ring buffer
or similar pattern"; reading R-RING).  The ring visits every
rank, so by the paper's invariant ("each ray will always find its respectively
closest intersection") the image, events and occlusion bits equal the union render; the
routing matrices and step counts have closed forms."""
import numpy as np
import pytest

import dpr_inputs as di
import oracle as orc

RING = 8


def _random_parts(seed, nranks, ntri=100, nsph=30):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1, 1, size=(ntri, 1, 3))
    v = (c + rng.uniform(-0.25, 0.25, size=(ntri, 3, 3))).astype(np.float32)
    sp = np.concatenate([rng.uniform(-1, 1, (nsph, 3)), rng.uniform(0.05, 0.2, (nsph, 1))], 1).astype(np.float32)
    tr, sr = rng.integers(0, nranks, ntri), rng.integers(0, nranks, nsph)
    parts = []
    for r in range(nranks):
        tv = v[tr == r].reshape(-1, 3)
        if tv.shape[0]:
            parts.append(di.Part(r, di.TRIS, albedo=(0.6, 0.5, 0.4), verts=tv,
                                 idx=np.arange(tv.shape[0], dtype=np.int32).reshape(-1, 3)))
        if (sr == r).any():
            parts.append(di.Part(r, di.SPHERES, albedo=(0.3, 0.7, 0.2), spheres=sp[sr == r]))
    return parts


def _frame(W, H, **kw):
    base = dict(W=W, H=H, spp=2, spp_batch=1, max_depth=3, ao_k=2, ao_radius=0.6,
                light_dir=di.f32(di.normalize((0.4, 1, -0.3))), E=(1, 1, 1), A=(0.3, 0.3, 0.3),
                B=(0.1, 0.1, 0.2), flags=RING)
    base.update(kw)
    return di.Frame(**base)


@pytest.mark.parametrize("nranks,seed", [(2, 0), (3, 1), (5, 2)])
def test_ring_equals_union_and_routing_closed_forms(nranks, seed):
    parts = _random_parts(seed, nranks)
    W, H = 24, 20
    cam = di.camera_basis((0.3, 0.8, -3.5), (0, 0, 0), (0, 1, 0), 45.0, W, H)
    fr = _frame(W, H)
    ring = orc.render(orc.OracleScene(parts, nranks), cam, fr, dp=True)
    u = orc.render(orc.OracleScene(di.union_parts(parts), 1), cam, fr)
    assert np.array_equal(ring.events, u.events) and np.array_equal(ring.occl, u.occl)
    assert np.array_equal(ring.gen, u.gen)
    assert np.allclose(ring.rgba, u.rgba, atol=1e-12, rtol=0)
    N = nranks
    prim = W * H * fr.spp
    # every ray is delivered to every rank exactly once
    for k in range(3):
        assert (ring.V[k] == ring.gen[k]).all()
    # all traffic is on the ring: rank a -> a+1 only
    off = np.ones((N, N), bool)
    off[np.arange(N), (np.arange(N) + 1) % N] = False
    assert (ring.S[:, off] == 0).all()
    # N-1 ring hops per ray, plus the send home of every child (path children = bounces)
    assert ring.S[0].sum() == ring.gen[0] * (N - 1) + (ring.gen[0] - prim)
    assert ring.S[1].sum() == ring.gen[1] * N
    assert ring.S[2].sum() == ring.gen[2] * N
    # the visit rule on the same partition: same image, fewer visits
    vr = orc.render(orc.OracleScene(parts, nranks), cam, _frame(W, H, flags=0), dp=True)
    assert np.array_equal(vr.events, ring.events) and vr.V.sum() < ring.V.sum()


def test_ring_steps_closed_form():
    """Camera inside a sphere: every path ray hits.  Depth 2 on N=3 ranks: primaries are
    traced in steps 0..2, their children (sent home) in 3..5, the bounce's children in 6..8:
    exactly 3N steps per batch, for every batch."""
    N = 3
    parts = [di.Part(r, di.SPHERES, albedo=(0.5, 0.5, 0.5), spheres=di.f32([[0, 0, 0, 5.0 + r]]))
             for r in range(N)]
    W = H = 12
    cam = di.camera_basis((0, 0, 0), (0, 0, 1), (0, 1, 0), 60.0, W, H)
    fr = _frame(W, H, spp=4, spp_batch=2, max_depth=2, ao_k=1, ao_radius=0.5)
    r = orc.render(orc.OracleScene(parts, N), cam, fr, dp=True)
    assert r.steps.tolist() == [3 * N, 3 * N]
    assert ((r.events[:, 0] & 0x80000000) == 0).all() and (r.events[:, 0] >= 2).all()
    # one rank: the ring degenerates to the plain renderer (no routing)
    one = orc.render(orc.OracleScene(di.union_parts(parts), 1), cam, fr, dp=True)
    assert (one.S == 0).all() and one.steps.tolist() == [3, 3]
    assert np.array_equal(one.events, r.events)
