"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and
bring its outputs back as numpy; run the oracle on the same seeded inputs."""
import numpy as np
import torch

import paper_2402_10128_b200 as G
from oracle import oracle as O


def settings_pair(rho=0.1, phi_mode=0, gaussian_only=0, background=(0.0, 0.0, 0.0), kernel=0):
    return (G.Settings(rho=rho, phi_mode=phi_mode, gaussian_only=gaussian_only, background=background, kernel=kernel),
            O.Settings(rho=rho, phi_mode=phi_mode, gaussian_only=gaussian_only, background=background,
                       kernel=kernel))


def gpu_forward(parts, cam, gs, pair_capacity=None, n_eval=True):
    P = parts.P
    dev = G.PlanarParams.from_inputs(parts)
    r = G.Renderer(P, cam.width, cam.height, pair_capacity=pair_capacity)
    ne = torch.zeros(cam.width * cam.height, dtype=torch.int32, device="cuda") if n_eval else None
    ncp = torch.zeros(cam.width * cam.height, dtype=torch.int32, device="cuda") if n_eval else None
    img = r.forward(dev, cam, gs, n_eval=ne, n_comp=ncp)
    torch.cuda.synchronize()
    f = r.frame
    cnt = f.counts()
    M = int(cnt.pairs)
    out = {
        "renderer": r, "params": dev, "counts": cnt, "image": img.cpu().numpy(),
        "depth": f.view("depth", torch.float32, P).cpu().numpy(),
        "pay0": f.view("pay0", torch.float32, 4 * P).cpu().numpy().reshape(P, 4),
        "pay1": f.view("pay1", torch.float32, 4 * P).cpu().numpy().reshape(P, 4),
        "pay2": f.view("pay2", torch.float32, P).cpu().numpy(),
        "radius": f.view("radius", torch.int32, P).cpu().numpy(),
        "rect": f.view("rect", torch.int16, 4 * P).cpu().numpy().view(np.uint16).reshape(P, 4).astype(np.int32),
        "status": f.view("status", torch.uint8, P).cpu().numpy().astype(np.int32),
        "flags": f.view("flags", torch.uint8, P).cpu().numpy().astype(np.int32),
        "ranges": f.ranges().cpu().numpy().view(np.uint32).astype(np.int64),
        "list": f.list(min(M, f.pair_capacity)).cpu().numpy().view(np.uint32).astype(np.int64) if M else np.zeros(0, np.int64),
        "final_T": f.view("final_T", torch.float32, cam.width * cam.height).cpu().numpy().reshape(cam.height, cam.width),
        "n_contrib": f.view("n_contrib", torch.int32, cam.width * cam.height).cpu().numpy().reshape(cam.height, cam.width),
    }
    if ne is not None:
        out["n_eval"] = ne.cpu().numpy().reshape(cam.height, cam.width)
        out["n_comp"] = ncp.cpu().numpy().reshape(cam.height, cam.width)
    return out


def gpu_backward(out, cam, gs, dL_dimage, accumulate=False, grads=None):
    r = out["renderer"]
    g = torch.from_numpy(np.ascontiguousarray(dL_dimage, np.float32)).cuda()
    grads = r.backward(out["params"], cam, gs, g, grads=grads, accumulate=accumulate)
    torch.cuda.synchronize()
    res = {}
    for n in G.PARAM_NAMES:
        res[n] = getattr(grads, n).cpu().numpy().astype(np.float64)
    return res, grads


def gpu_keys(out):
    """Reconstruct (tile << 32 | depth bits) keys of the GPU's sorted lists."""
    ranges, lst = out["ranges"], out["list"]
    tiles = np.repeat(np.arange(ranges.size - 1, dtype=np.uint64), np.diff(ranges))
    db = out["depth"].view(np.uint32).astype(np.uint64)
    return (tiles << np.uint64(32)) | db[lst]


def ambiguous_particles(pre, amb_pixels, tiles_x):
    """Particles whose rect covers a tile that holds an ambiguous pixel."""
    ys, xs = np.nonzero(amb_pixels)
    bad = np.zeros(pre["status"].size, bool)
    if ys.size == 0:
        return bad
    tset = set(zip((ys // 16).tolist(), (xs // 16).tolist()))
    x0, y0, x1, y1 = pre["rect"]
    vis = pre["status"] == 0
    for (ty, tx) in tset:
        bad |= vis & (x0 <= tx) & (tx < x1) & (y0 <= ty) & (ty < y1)
    return bad


def grad_mismatch(ga, gr, rel=1e-3, floor=1e-6):
    """north_star: |g_gpu - g_ref| <= max(rel |g_ref|, floor)."""
    return np.abs(ga - gr) > np.maximum(rel * np.abs(gr), floor)
