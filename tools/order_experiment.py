"""Experiment: stage times of the bench step (config 3) with the particles stored in
their generated (random) order vs in Morton order of their means."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ges_inputs as gi  # noqa: E402
import paper_2402_10128_b200 as G  # noqa: E402


def morton_perm(mean):
    lo, hi = mean.min(axis=1, keepdims=True), mean.max(axis=1, keepdims=True)
    q = np.clip(((mean - lo) / (hi - lo + 1e-30) * 1023).astype(np.int64), 0, 1023)

    def spread(x):
        x = (x | (x << 16)) & 0x030000FF
        x = (x | (x << 8)) & 0x0300F00F
        x = (x | (x << 4)) & 0x030C30C3
        x = (x | (x << 2)) & 0x09249249
        return x
    code = spread(q[0]) | (spread(q[1]) << 1) | (spread(q[2]) << 2)
    return np.argsort(code, kind="stable")


def run(parts, cam, label, steps=30):
    params = G.PlanarParams.from_inputs(parts)
    P = params.P
    st = G.Settings(rho=0.1)
    r = G.Renderer(P, cam.width, cam.height)
    img = r.forward(params, cam, st)
    r.grow(int(r.frame.counts().slots))
    dL = torch.from_numpy(gi.upstream_grad(1003, 0, cam.width, cam.height)).cuda()
    grads = G.PlanarParams.zeros(P, params.sh_degree)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    names = ["preprocess", "sort", "fwd", "bwd_tiles", "bwd_particles"]
    acc = np.zeros(5)
    for it in range(steps + 3):
        flush.fill_(1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        G.ges_preprocess(params, cam, st, r.frame); ev[1].record()
        G.ges_sort(r.frame); ev[2].record()
        G.ges_render_fwd(r.frame, st, img); ev[3].record()
        G.ges_render_bwd_tiles(st, r.frame, dL); ev[4].record()
        G.ges_backward_particles(params, cam, st, r.frame, grads); ev[5].record()
        ev[5].synchronize()
        if it >= 3:
            acc += [ev[k].elapsed_time(ev[k + 1]) for k in range(5)]
    acc /= steps
    print(label, " ".join(f"{n} {1e3 * v:.1f}" for n, v in zip(names, acc)), f"total {1e3 * acc.sum():.1f} us")


sc = gi.make_config(3)
cam = sc.cameras[0]
run(sc.particles, cam, "index order ")
perm = morton_perm(sc.particles.mean.astype(np.float64))
run(sc.particles.subset(perm), cam, "morton order")
