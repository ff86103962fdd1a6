import os, sys, json
sys.path.insert(0, os.getcwd())
from bench import make_scene
from paper_2407_00179_b200 import dpr
import torch
sc = make_scene("c3", 1)
d = dpr.Device.create(0, 1, 0)
d.commit_scene_parts(sc.parts); d.commit_world(); d.set_camera(sc.camera); d.set_frame(sc.frame)
for i in range(3):
    d.render_frame()
st = d.get_stats()
print(json.dumps({k: (st[k].tolist() if hasattr(st[k], 'tolist') else st[k]) for k in ("ms_frame", "vol_samples_local", "kernel_vols_local", "kernel_launches_local")}))
d.release()
