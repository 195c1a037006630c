"""Probe: an 8-view fwd+bwd iteration with the views on two streams (two frames; the
S5b accumulations into the one gradient buffer serialised by events) against one stream.
python tools/two_stream_probe.py [config]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import ges_inputs as gi
import paper_2402_10128_b200 as G

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scene = gi.make_config(cfg)
cams = scene.cameras[:8] if cfg == 2 else [scene.cameras[k] for k in
                                           np.random.default_rng(2402).choice(len(scene.cameras), 8, replace=False)]
params = G.PlanarParams.from_inputs(scene.particles)
st = G.Settings(rho=scene.rho)
W, H = cams[0].width, cams[0].height
P = params.P
grads = G.PlanarParams.zeros(P, params.sh_degree)
rs = [G.Renderer(P, W, H) for _ in range(2)]
imgs = [torch.empty((3, H, W), device="cuda") for _ in range(2)]
dLs = [torch.from_numpy(gi.upstream_grad(scene.seed, k, W, H)).cuda() for k in range(8)]
for r in rs:
    for c in cams:
        r.forward(params, c, st)
        r.grow(int(r.frame.counts().slots))
torch.cuda.synchronize()
s0 = torch.cuda.Stream()
s1 = torch.cuda.Stream()


def one_stream(s):
    f = rs[0].frame
    for k, c in enumerate(cams):
        G.ges_preprocess(params, c, st, f, s)
        G.ges_sort(f, s)
        G.ges_render_fwd(f, st, imgs[0], None, s)
        G.ges_render_bwd(params, c, st, f, dLs[k], grads, k > 0, s)


def two_streams(s):
    ss = [s, s1]
    s1.wait_stream(s)
    ev_b = None
    for k, c in enumerate(cams):
        q = ss[k % 2]
        f = rs[k % 2].frame
        G.ges_preprocess(params, c, st, f, q)
        G.ges_sort(f, q)
        G.ges_render_fwd(f, st, imgs[k % 2], None, q)
        G.ges_render_bwd_tiles(st, f, dLs[k], q)
        if ev_b is not None:
            q.wait_event(ev_b)          # S5b accumulations in view order, never concurrent
        G.ges_backward_particles(params, c, st, f, grads, k > 0, q)
        ev_b = torch.cuda.Event()
        ev_b.record(q)
    s.wait_stream(s1)


def time_graph(fn, reps=20):
    g = torch.cuda.CUDAGraph()
    s0.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s0):
        fn(s0)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


one_stream(torch.cuda.current_stream())
torch.cuda.synchronize()
ref = grads.flat.clone()
two_streams(torch.cuda.current_stream())
torch.cuda.synchronize()
diff = float(((grads.flat - ref).abs().max() / ref.abs().max()).item())
t1 = time_graph(one_stream)
t2 = time_graph(two_streams)
print(f"config {cfg}: one stream {t1:.3f} ms, two streams {t2:.3f} ms per 8-view iteration "
      f"({t1 / t2:.3f}x); max rel grad diff {diff:.2e}")
