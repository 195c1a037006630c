"""Depth-sort rank-phase timings (needs a GES_DS_TIMING=3 build: python paper_2402_10128_b200/_build.py
--variant dst3 -DGES_DS_TIMING=3 [-DGES_DS_TIMING_SHIFT=18]; run with GES_LIB=.../dst3/libges.so)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import ges_inputs as gi
import paper_2402_10128_b200 as G
from paper_2402_10128_b200 import _lib as L
sc = gi.make_config(3); cam = sc.cameras[0]
params = G.PlanarParams.from_inputs(sc.particles); st = G.Settings(rho=sc.rho)
r = G.Renderer(params.P, cam.width, cam.height)
r.forward(params, cam, st)
for _ in range(3):
    G.ges_preprocess(params, cam, st, r.frame); G.ges_sort(r.frame)
torch.cuda.synchronize()
t = (C.c_ulonglong * 8)()
L.load().ges_debug_ds_times(t)
a = np.array(list(t)[:5], dtype=np.int64)
print("pass-1 rank phases us (load, match loop, over-warps+scan512, smem scatter):", np.round(np.diff(a) / 1e3, 2))
print("warp 0 cycles: peers", t[5], "serial updates", t[6])
