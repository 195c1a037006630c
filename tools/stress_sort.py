"""Stress of the sort/binning protocols (tickets, published words, look-backs):
N frames of config 3 (and config 4's first camera) through ges_preprocess + ges_sort,
every list and range compared with the first frame's (they are bit-exact by design).
Usage: python tools/stress_sort.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ges_inputs as gi  # noqa: E402
import paper_2402_10128_b200 as G  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for cfg, kw in ((3, {}), (4, {"n_views": 1}), (2, {})):
    sc = gi.make_config(cfg, **kw)
    cam = sc.cameras[0]
    params = G.PlanarParams.from_inputs(sc.particles)
    st = G.Settings(rho=sc.rho)
    r = G.Renderer(params.P, cam.width, cam.height)
    r.forward(params, cam, st)
    r.grow(int(r.frame.counts().slots))
    G.ges_preprocess(params, cam, st, r.frame)
    G.ges_sort(r.frame)
    torch.cuda.synchronize()
    M = int(r.frame.counts().pairs)
    ref_list, ref_rng = r.frame.list(M).clone(), r.frame.ranges().clone()
    bad = 0
    for it in range(N):
        G.ges_preprocess(params, cam, st, r.frame)
        G.ges_sort(r.frame)
        if it % 10 == 9:
            torch.cuda.synchronize()
            if int(r.frame.counts().pairs) != M or not torch.equal(r.frame.list(M), ref_list) or \
                    not torch.equal(r.frame.ranges(), ref_rng):
                bad += 1
    torch.cuda.synchronize()
    print(f"config {cfg}: {N} frames, {N // 10} compared, {bad} differing; M = {M}")
    assert bad == 0
