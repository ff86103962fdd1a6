import sys
import numpy as np
sys.path.insert(0, '.')
import dpr_inputs as di
import oracle as orc
sc = di.config4(nranks=1, n_clusters=24, per_cluster=400, G=41, W=72, H=40, spp=2)
pix = np.array([1254, 2350], np.int64)
osc = orc.OracleScene(sc.parts, 1)
fr = di.Frame(**sc.frame.__dict__)
a = orc.render(osc, sc.camera, fr, pixels=pix)
orc.set_brute(True)
b = orc.render(osc, sc.camera, fr, pixels=pix)
orc.set_brute(False)
for i, p in enumerate(pix):
    for s in range(2):
        print(p, s, "bvh", [hex(x) for x in a.events[s, :, i]], "brute", [hex(x) for x in b.events[s, :, i]])
