"""Small renders through every kernel family, for compute-sanitizer (memcheck / racecheck)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dpr_inputs as di  # noqa: E402
from tests.gpu_helpers import gpu_render  # noqa: E402


def vol(G=17, nb=2, nr=2):
    field = di.volume_field(G)
    tf = di.default_tf(alpha_max=0.3, s0=0.2)
    h = np.float32(2.0 / (G - 1))
    parts = []
    for r, (lo, hi) in enumerate(di.brick_boxes((G - 1,) * 3, nb)):
        vox = field[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
        parts.append(di.Part(r % nr, di.BRICK, gdims=(G,) * 3, origin=(-1, -1, -1), spacing=(float(h),) * 3,
                             cell_lo=lo, cell_hi=hi, voxels=np.ascontiguousarray(vox), tf=tf))
    return parts, float(h)


sc = di.config1()
gpu_render(sc.parts, 2, sc.camera, sc.frame)
s2 = di.config2(nranks=2, G=17, W=24, H=20, spp=2, spp_batch=2)
gpu_render(s2.parts, 2, s2.camera, s2.frame)
gpu_render(di.union_parts(s2.parts), 1, s2.camera, s2.frame)
parts, h = vol()
cam = di.camera_basis((0.3, 1.5, -3.0), (0, -0.2, 0), (0, 1, 0), 50.0, 16, 16)
for flags in (0, 8, 16, 24):
    fr = di.Frame(W=16, H=16, spp=2, spp_batch=1, max_depth=2, ao_k=1, ao_radius=0.3, dt=h,
                  light_dir=di.f32(di.normalize((0.2, 1, 0.1))), E=(1, 1, 1), A=(0.2, 0.2, 0.2), flags=flags)
    gpu_render(parts + s2.parts, 2, cam, fr)
os.environ["DPR_EXCHANGE"] = "fused"
gpu_render(s2.parts, 2, s2.camera, s2.frame)
print("sanitize run ok")
