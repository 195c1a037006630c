"""Per-tile start/end times of S4 and S5a and their tails under different launch orders
(needs a GES_TILE_CLOCK=1 build: python paper_2402_10128_b200/_build.py --variant clk
-DGES_TILE_CLOCK=1; run with GES_LIB=paper_2402_10128_b200/build/variants/clk/libges.so).
Prints the kernel span, how many CTAs are busy over time, and the span when the tiles
are launched heaviest-first by several cost predictors."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import ges_inputs as gi
import paper_2402_10128_b200 as G
from paper_2402_10128_b200 import _lib as L

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sc = gi.make_config(cfg)
cam = sc.cameras[0]
params = G.PlanarParams.from_inputs(sc.particles)
st = G.Settings(rho=sc.rho)
r = G.Renderer(params.P, cam.width, cam.height)
img = r.forward(params, cam, st)
dL = torch.from_numpy(gi.upstream_grad(sc.seed, 0, cam.width, cam.height)).cuda()
grads = r.backward(params, cam, st, dL)
torch.cuda.synchronize()
lib = L.load()
buf = (C.c_ulonglong * (2 * 16384 * 3))()
T = r.frame.c.tiles_x * r.frame.c.tiles_y
tx = r.frame.c.tiles_x
W, H = cam.width, cam.height


def run(order_fwd=None, order_bwd=None, reps=5):
    for w, o in ((0, order_fwd), (1, order_bwd)):
        if o is None:
            lib.ges_debug_tile_order(w, None, 0)
        else:
            arr = np.ascontiguousarray(o, np.int32)
            lib.ges_debug_tile_order(w, arr.ctypes.data_as(C.c_void_p), int(arr.size))
    spans, res = [], None
    for _ in range(reps):
        lib.ges_debug_tile_clock(buf, 1)
        G.ges_preprocess(params, cam, st, r.frame)
        G.ges_sort(r.frame)
        G.ges_render_fwd(r.frame, st, img)
        G.ges_render_bwd(params, cam, st, r.frame, dL, grads)
        torch.cuda.synchronize()
        lib.ges_debug_tile_clock(buf, 0)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 16384, 3)[:, :T].astype(np.int64).copy()
        spans.append([(a[w, :, 1].max() - a[w, :, 0].min()) / 1e3 for w in range(2)])
        res = a
    lib.ges_debug_tile_order(0, None, 0)
    lib.ges_debug_tile_order(1, None, 0)
    return np.median(np.array(spans), axis=0), res


base, a = run()
ranges = r.frame.view("ranges", torch.int32, T + 1).cpu().numpy().astype(np.int64)
lens = np.diff(ranges)
nc = r.frame.view("n_contrib", torch.int32, W * H).cpu().numpy().astype(np.int64).reshape(H, W)
ncp = np.zeros((r.frame.c.tiles_y * 16, tx * 16), np.int64)
ncp[:H, :W] = nc
t4 = ncp.reshape(r.frame.c.tiles_y, 16, tx, 16)
nc_sum = t4.sum(axis=(1, 3)).reshape(-1)[:T]
# backward warps: 8 x 16 regions (left / right half of the tile), walk extent = max n_contrib
halves = t4.reshape(r.frame.c.tiles_y, 16, tx, 2, 8).max(axis=(1, 4))
nc_wmax = halves.sum(axis=-1).reshape(-1)[:T]
nc_hmax = halves.max(axis=-1).reshape(-1)[:T]
nc_tmax = t4.max(axis=(1, 3)).reshape(-1)[:T]
for w, name in enumerate(["render_fwd", "render_bwd"]):
    s = a[w, :, 0] - a[w, :, 0].min()
    e = a[w, :, 1] - a[w, :, 0].min()
    d = e - s
    span = e.max()
    nb = int(span // 1000) + 1
    act = np.zeros(nb + 1)
    np.add.at(act, s // 1000, 1)
    np.add.at(act, e // 1000, -1)
    act = np.cumsum(act)[:nb]
    print(f"{name}: span {span/1e3:.1f} us (median of 5: {base[w]:.1f}), mean tile {d.mean()/1e3:.1f} us, "
          f"max {d.max()/1e3:.1f}; {d.sum()/span:.0f} CTAs busy on average (peak {act.max():.0f}); "
          f"last tile start {s.max()/1e3:.1f} us")
    print("  busy CTAs per 10 us:", " ".join(f"{int(x)}" for x in act[::10]))
    for pname, pv in (("list length", lens), ("sum n_contrib", nc_sum), ("warp max n_contrib", nc_wmax),
                      ("max of the halves", nc_hmax)):
        print(f"  corr(duration, {pname}) {np.corrcoef(d, pv)[0, 1]:.3f}")
d_f = a[0, :, 1] - a[0, :, 0]
best_c, best_r = None, -2
for c in (50, 100, 200, 300, 400, 600, 800, 1200, 1600):
    rr = np.corrcoef(d_f, np.minimum(lens, c))[0, 1]
    print(f"corr(fwd duration, min(list length, {c})) {rr:.3f}")
    if rr > best_r:
        best_c, best_r = c, rr
capped = np.minimum(lens, best_c)
d_b = a[1, :, 1] - a[1, :, 0]
print(f"corr(fwd duration, bwd duration) {np.corrcoef(d_f, d_b)[0, 1]:.3f}")
experiments = {
    "measured durations (bound)": (np.argsort(-d_f, kind="stable"), np.argsort(-d_b, kind="stable")),
    "list length": (np.argsort(-lens, kind="stable"), np.argsort(-lens, kind="stable")),
    "sum n_contrib": (np.argsort(-nc_sum, kind="stable"), np.argsort(-nc_sum, kind="stable")),
    "warp max n_contrib": (np.argsort(-nc_wmax, kind="stable"), np.argsort(-nc_wmax, kind="stable")),
    "max of the halves": (np.argsort(-nc_hmax, kind="stable"), np.argsort(-nc_hmax, kind="stable")),
    "sum + max halves": (np.argsort(-(nc_wmax + nc_hmax), kind="stable"), np.argsort(-(nc_wmax + nc_hmax), kind="stable")),
    "bwd by fwd duration": (None, np.argsort(-d_f, kind="stable")),
    "fwd by capped list length": (np.argsort(-capped, kind="stable"), None),
}
print(f"natural order: fwd {base[0]:.1f} us, bwd {base[1]:.1f} us")
for k, (of, ob) in experiments.items():
    sp, _ = run(of, ob)
    print(f"heaviest first by {k}: fwd {sp[0]:.1f} us, bwd {sp[1]:.1f} us")
