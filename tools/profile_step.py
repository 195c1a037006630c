"""Runs `--steps` fwd+bwd steps of the bench workload (config 3) for profilers
(ncu / compute-sanitizer).  No timing; no oracle."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import ges_inputs as gi  # noqa: E402
import paper_2402_10128_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--P", type=int, default=None)
args = ap.parse_args()
sc = gi.make_config(args.config, P=args.P)
cam = sc.cameras[0]
params = G.PlanarParams.from_inputs(sc.particles)
st = G.Settings(rho=sc.rho)
r = G.Renderer(params.P, cam.width, cam.height)
img = r.forward(params, cam, st)
r.grow(int(r.frame.counts().slots))
dL = torch.from_numpy(gi.upstream_grad(sc.seed, 0, cam.width, cam.height)).cuda()
grads = G.PlanarParams.zeros(params.P, params.sh_degree)
for _ in range(args.steps):
    G.ges_preprocess(params, cam, st, r.frame)
    G.ges_sort(r.frame)
    G.ges_render_fwd(r.frame, st, img)
    G.ges_render_bwd(params, cam, st, r.frame, dL, grads)
torch.cuda.synchronize()
c = r.frame.counts()
print(f"ok visible={c.visible} pairs={c.pairs} overflow={c.overflow}")
