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
ctr = r.frame.view("counters", torch.int64, 16).cpu().tolist()
t = ctr[8:16]
names = ["key range", "pass 0", "pass 1", "pass 2", "pass 3/none", "items sum", "items scan"]
for i, n in enumerate(names):
    if t[i + 1] >= t[i] > 0:
        print(f"{n:12s} {(t[i + 1] - t[i]) / 1e3:8.2f} us")
print(f"total        {(t[7] - t[0]) / 1e3:8.2f} us")
