"""Per-stage device times (CUDA events, median of N) of the bench workload.
Usage: python tools/stage_times.py [--config 3] [--steps 20]"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import ges_inputs as gi  # noqa: E402
import paper_2402_10128_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--tag", default="")
ap.add_argument("--P", type=int, default=None, help="particle count override (config 3's distributions)")
args = ap.parse_args()
sc = gi.make_config(args.config, **({"P": args.P} if args.P else {}))
cam = sc.cameras[0]
params = G.PlanarParams.from_inputs(sc.particles)
st = G.Settings(rho=sc.rho)
r = G.Renderer(params.P, cam.width, cam.height)
img = r.forward(params, cam, st)
r.grow(int(r.frame.counts().slots))
dL = torch.from_numpy(gi.upstream_grad(sc.seed, 0, cam.width, cam.height)).cuda()
grads = G.PlanarParams.zeros(params.P, params.sh_degree)
names = ["preprocess", "sort", "render_fwd", "render_bwd_tiles", "backward_particles"]
acc = {n: [] for n in names}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(args.steps + 3):
    flush.fill_(1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    G.ges_preprocess(params, cam, st, r.frame)
    ev[1].record()
    G.ges_sort(r.frame)
    ev[2].record()
    G.ges_render_fwd(r.frame, st, img)
    ev[3].record()
    G.ges_render_bwd_tiles(st, r.frame, dL)
    ev[4].record()
    G.ges_backward_particles(params, cam, st, r.frame, grads)
    ev[5].record()
    ev[5].synchronize()
    if it >= 3:
        for i, n in enumerate(names):
            acc[n].append(ev[i].elapsed_time(ev[i + 1]))
res = {n: round(statistics.median(v), 4) for n, v in acc.items()}
res["total"] = round(sum(res.values()), 4)
print(json.dumps({"tag": args.tag, "env": {k: v for k, v in os.environ.items() if k.startswith("GES_")}, **res}))
