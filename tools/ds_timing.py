"""Phase timings of the cooperative depth sort (needs a GES_DS_TIMING build:
python paper_2402_10128_b200/_build.py --variant dstime -DGES_DS_TIMING=1; GES_LIB=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ges_inputs as gi  # noqa: E402
import paper_2402_10128_b200 as G  # noqa: E402

sc = gi.make_config(3)
cam = sc.cameras[0]
params = G.PlanarParams.from_inputs(sc.particles)
st = G.Settings(rho=sc.rho)
r = G.Renderer(params.P, cam.width, cam.height)
r.forward(params, cam, st)
r.grow(int(r.frame.counts().slots))
for _ in range(5):
    G.ges_preprocess(params, cam, st, r.frame)
    G.ges_sort(r.frame)
torch.cuda.synchronize()
ctr = r.frame.view("counters", torch.int64, 24).cpu().tolist()
t = ctr[16:24]
# slots: 0 start, 1 after phase H, 2 / 3 after passes 0 / 1 (non-last), 4 last pass hist done,
# 5 last pass prefix done, 6 end
names = [("phase H", 0, 1), ("pass 0", 1, 2), ("pass 1", 2, 3), ("last hist", 3, 4), ("last prefix", 4, 5),
         ("last scatter", 5, 6), ("total", 0, 6)]
for n, i, j in names:
    if t[j] >= t[i] > 0:
        print(f"{n:12s} {(t[j] - t[i]) / 1e3:8.2f} us")
