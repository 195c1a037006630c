"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel of the hot path on configs 0 and 1 -- S1, the depth sort,
the binning, S4, S5a, S5b -- the exact-beta kernel, screen-tile bands, the loss
front end and Adam.  Exits 0 after checking the images against the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [--small]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ges_inputs as gi  # noqa: E402
import paper_2402_10128_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--small", action="store_true", help="config 1 at 5,000 particles (racecheck is slow)")
args = ap.parse_args()


def case(cfg, kernel=0, band=None, **kw):
    sc = gi.make_config(cfg, **kw)
    cam = sc.cameras[0]
    params = G.PlanarParams.from_inputs(sc.particles)
    st = G.Settings(rho=sc.rho, kernel=kernel)
    if band is not None:
        st = G.Settings(rho=sc.rho, kernel=kernel, tile_row_begin=band[0], tile_row_step=band[1])
    r = G.Renderer(params.P, cam.width, cam.height)
    img = r.forward(params, cam, st)
    dL = torch.from_numpy(gi.upstream_grad(sc.seed, 0, cam.width, cam.height)).cuda()
    grads = r.backward(params, cam, st, dL)
    torch.cuda.synchronize()
    if band is None:
        ref = O.render(sc.particles, cam, O.Settings(rho=sc.rho, kernel=kernel))
        d = np.abs(img.cpu().numpy() - ref["image"])
        d[:, ref["amb"] != 0] = 0
        assert d.max() <= 1e-4, (cfg, kernel, d.max())
    assert torch.isfinite(grads.flat).all()
    return params, grads, img, cam


P1 = 5000 if args.small else None
case(0)
case(0, kernel=1)
case(1, beta_value=2.0, P=P1)
case(1, beta_value=0.5, P=P1, kernel=1)
case(0, band=(1, 3))
params, grads, img, cam = case(0)
loss = G.Loss(cam.width, cam.height)
gt = torch.rand_like(img)
mask = loss.mask(gt, 0.75)
loss(img, gt, mask)
G.Adam(params).step(params, grads)
torch.cuda.synchronize()
print("sanitize cases ok")
