"""Commit one configuration's parts and rebuild the world K times (profiling the LBVH build,
row a1, in isolation): python tools/build_only.py [c2|c4|c5] [K]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import make_scene  # noqa: E402
from paper_2407_00179_b200 import dpr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sc = make_scene(cfg, 1)
dev = dpr.Device.create(0, 1, 0)
for p in sc.parts:
    dev.commit_part(p)
ms = []
for _ in range(K):
    dev.commit_world()
    ms.append(dev.get_stats()["ms_build"])
torch.cuda.synchronize()
print(json.dumps({"config": cfg, "ms_build": ms, "prims": int(sum(p.nprims() for p in sc.parts))}))
dev.release()
