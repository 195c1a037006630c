"""Binning emission-trip counts and direct-path chunks (needs a GES_BIN_STATS=1 build; run with
GES_LIB=paper_2402_10128_b200/build/variants/stats/libges.so)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
import ges_inputs as gi
import paper_2402_10128_b200 as G
from paper_2402_10128_b200 import _lib as L
sc = gi.make_config(3); cam = sc.cameras[0]
params = G.PlanarParams.from_inputs(sc.particles); st = G.Settings(rho=sc.rho)
r = G.Renderer(params.P, cam.width, cam.height)
r.forward(params, cam, st); torch.cuda.synchronize()
lib = L.load()
if hasattr(lib, "ges_debug_bin_trips"):
    out = (C.c_ulonglong * 6)()
    lib.ges_debug_bin_trips(out)
    a = list(out)
    G.ges_preprocess(params, cam, st, r.frame); G.ges_sort(r.frame); torch.cuda.synchronize()
    lib.ges_debug_bin_trips(out)
    b = list(out)
    c = r.frame.counts()
    print("trips rows", b[0]-a[0], "cols", b[1]-a[1], "pairs", c.pairs, "pairs/trip", c.pairs/(b[1]-a[1]))
    print("direct-path chunks: rows", b[2]-a[2], "of", b[3]-a[3], " cols", b[4]-a[4], "of", b[5]-a[5])
    sys.exit(0)
import numpy as np
t = (C.c_ulonglong * 512)(); n = C.c_int(0)
lib.ges_debug_bin_times(t, C.byref(n))
for _ in range(3):
    G.ges_preprocess(params, cam, st, r.frame); G.ges_sort(r.frame)
torch.cuda.synchronize()
lib.ges_debug_bin_times(t, C.byref(n))
a = np.array(list(t), dtype=np.int64).reshape(64, 8)[:n.value, :7]
print("chunks of CTA 0:", n.value)
d = np.diff(a, axis=1) / 1e3
print("phase us (ticket, load+count, excl+scans, emission, copy, sync) per chunk:")
for row in d[: n.value]:
    print(" ", np.round(row, 2), " gap to next:", )
if n.value > 1:
    print("chunk period us:", np.round(np.diff(a[:, 0]) / 1e3, 2))
