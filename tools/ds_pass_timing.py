"""Depth-sort per-pass phase times of CTA 0 and of the last CTA (needs a GES_DS_TIMING=4
build: python paper_2402_10128_b200/_build.py --variant dst4 -DGES_DS_TIMING=4; run with
GES_LIB=paper_2402_10128_b200/build/variants/dst4/libges.so)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import ges_inputs as gi
import paper_2402_10128_b200 as G
from paper_2402_10128_b200 import _lib as L

sc = gi.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
cam = sc.cameras[0]
params = G.PlanarParams.from_inputs(sc.particles)
st = G.Settings(rho=sc.rho)
r = G.Renderer(params.P, cam.width, cam.height)
r.forward(params, cam, st)
res = []
for _ in range(5):
    G.ges_preprocess(params, cam, st, r.frame)
    G.ges_sort(r.frame)
    torch.cuda.synchronize()
    t = (C.c_ulonglong * 40)()
    L.load().ges_debug_ds_pass_times(t)
    res.append(np.array(list(t), dtype=np.int64).reshape(2, 4, 5))
a = np.median(np.stack(res), axis=0)
t0 = a[0, 0, 0]
for p in range(4):
    if a[0, p, 0] == 0 or a[0, p, 0] < t0:
        continue
    for c, name in ((0, "CTA 0"), (1, "last CTA")):
        x = a[c, p]
        d = np.diff(x) / 1e3
        print(f"pass {p} {name:8s}: start {(x[0] - t0) / 1e3:6.2f} us; rank {d[0]:5.2f}, prefix {d[1]:5.2f}, "
              f"write {d[2]:5.2f}, barrier {d[3]:5.2f}")
