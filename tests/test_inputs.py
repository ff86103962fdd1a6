"""Synthetic input generators (dpr_inputs): shapes and determinism of the workloads
(SURVEY 8(d) 'Concrete synthetic inputs'); oracle BVH vs brute force on the C2 mesh
family."""
import numpy as np

import dpr_inputs as di
import oracle as orc


def test_gyroid_count_scaling_and_determinism():
    """C2 mesh: marching-tetrahedra gyroid; ~110*G^2 triangles, bit-identical across
    thread counts (order is z-major regardless of the split)."""
    v1, i1 = di.gyroid_mesh(41, nthreads=1)
    v2, i2 = di.gyroid_mesh(41, nthreads=5)
    assert np.array_equal(v1, v2) and np.array_equal(i1, i2)
    n = i1.shape[0]
    assert 0.8 * 110 * 41 ** 2 < n < 1.2 * 110 * 41 ** 2
    assert np.abs(v1).max() <= 1.0 + 1e-6
    tri = v1[i1].astype(np.float64)
    area = np.linalg.norm(np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]), axis=1)
    assert (area > 0).all()


def test_gyroid_indexed_mesh_is_welded_manifold():
    """One shared vertex per cut grid edge: ~T/2 vertices, every mesh edge used by at most
    two triangles and almost all (all but the domain boundary / dropped slivers) by two."""
    v, i = di.gyroid_mesh(41)
    assert i.min() >= 0 and i.max() < v.shape[0]
    assert 0.45 < v.shape[0] / i.shape[0] < 0.6
    e = np.sort(np.concatenate([i[:, [0, 1]], i[:, [1, 2]], i[:, [2, 0]]]), axis=1)
    _, c = np.unique(e, axis=0, return_counts=True)
    assert c.max() == 2 and (c == 2).mean() > 0.9
    # the split keeps the geometry: the parts' triangles are exactly the mesh's triangles
    parts = di.split_mesh(v, i, 3, (1, 1, 1))
    got = np.concatenate([p.verts[p.idx].reshape(-1, 9) for p in parts])
    ref = v[i].reshape(-1, 9)
    key = lambda a: a[np.lexsort(a.T[::-1])]
    assert np.array_equal(key(got), key(ref))


def test_bisect_partition_balanced():
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1, 1, (1000, 3))
    for n in (1, 2, 3, 4, 8):
        g = di.bisect_partition(pts, n)
        c = np.bincount(g, minlength=n)
        assert c.sum() == 1000 and c.max() - c.min() <= 2


def test_brick_boxes_tile_domain():
    for n in (1, 2, 3, 4, 8):
        boxes = di.brick_boxes((16, 16, 16), n)
        vol = sum(np.prod(np.subtract(hi, lo)) for lo, hi in boxes)
        assert len(boxes) == n and vol == 16 ** 3


def test_camera_basis_orthogonal():
    c = di.camera_basis((2.2, 1.6, 2.8), (0, 0, 0), (0, 1, 0), 45.0, 1024, 512)
    U, V = c.U.astype(np.float64), c.V.astype(np.float64)
    assert abs(U @ V) < 1e-6
    assert abs(np.linalg.norm(U) / np.linalg.norm(V) - 2.0) < 1e-6


def test_oracle_bvh_on_gyroid_equals_brute_force():
    """P9 on the C2 mesh family (~27k triangles): oracle BVH closest == brute force on 400
    camera-like rays through the mesh."""
    v, i = di.gyroid_mesh(17)
    sc = orc.OracleScene([di.Part(0, di.TRIS, verts=v, idx=i)], 1)
    rng = np.random.default_rng(5)
    o = np.array([2.2, 1.6, 2.8], np.float32)
    for k in range(400):
        tgt = rng.uniform(-1, 1, 3)
        d = (tgt - o) / np.linalg.norm(tgt - o)
        d = d.astype(np.float32)
        assert sc.closest(o, d, brute=True) == sc.closest(o, d)
