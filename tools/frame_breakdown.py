"""Per-phase device times of one configs[1] frame from dpr_get_stats (library CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dpr_inputs as di  # noqa: E402
from paper_2407_00179_b200 import dpr  # noqa: E402

sc = di.config2(nranks=1)
dev = dpr.Device.create(0, 1, 0)
for p in sc.parts:
    dev.commit_part(p)
dev.commit_world()
dev.set_camera(sc.camera)
dev.set_frame(sc.frame)
for _ in range(3):
    dev.commit_world()
    dev.render_frame()
torch.cuda.synchronize()
acc = {}
for _ in range(5):
    dev.commit_world()
    dev.render_frame()
    st = dev.get_stats()
    for k in ("ms_frame", "ms_build", "ms_gen", "ms_trace_path", "ms_trace_occl", "ms_exchange", "ms_reduce"):
        acc[k] = acc.get(k, 0.0) + st[k] / 5
known = acc["ms_gen"] + acc["ms_trace_path"] + acc["ms_trace_occl"] + acc["ms_exchange"] + acc["ms_reduce"]
for k, v in acc.items():
    print(f"{k:16s} {v:8.3f} ms")
print(f"{'frame - listed':16s} {acc['ms_frame'] - known:8.3f} ms  (shade + resolve + host gaps)")
dev.release()
