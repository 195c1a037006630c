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


def grad_mismatch(ga, gr, rel=1e-3, floor=1e-6):
    """north_star: |g_gpu - g_ref| <= max(rel |g_ref|, floor)."""
    return np.abs(ga - gr) > np.maximum(rel * np.abs(gr), floor)


# R19: an fp32 evaluation of a gradient entry is accurate to about
# R19_C * 2^-24 * round + sens, with round / sens the oracle's first-order error
# scales of the entry (oracle.grad_error_scale: the rounding of the sums and
# products, and the propagated fp32 error of the forward alphas and
# transmittances).  R19_C = 8 (per-term rounding: ex2.approx 2 ulp, rcp.approx
# 1 ulp, ~5 roundings) + 24 (reduction depth: 5 SHFL levels, <= 19 levels of
# atomics and partial sums).
EPS32 = 2.0 ** -24
R19_C = 32.0


def masked_upstream(dL, amb):
    """dL/dimage with the oracle-flagged threshold-ambiguous pixels (R18) zeroed.
    Every S5a term is linear in its pixel's dL/dC (and dL/dC . bg), so those
    pixels drop out of both sides exactly and every particle can be compared."""
    d = np.array(dL, np.float32, copy=True)
    d[:, amb != 0] = 0.0
    return d


def oracle_grads(parts, cam, osx, pre, dL, offsets=None, lst=None):
    """The oracle's S5 gradients and the R19 error scale of every entry."""
    if offsets is None:
        offsets, lst = O.tile_lists(pre)
    g2d, gmag = O.render_bwd(pre, cam, osx, offsets, lst, dL, with_abs=True)
    grads = O.backward_particles(parts, cam, osx, g2d, pre["status"], pre["flags"])
    scale = O.grad_error_scale(parts, cam, osx, g2d, gmag, pre["status"], pre["flags"])
    return grads, scale


def check_grads(gg, ref, scale, status, label=""):
    """Every visible particle's gradient entries against the oracle:
    |g_gpu - g_ref| <= max(1e-3 |g_ref|, 1e-6)  (north_star), or, for entries
    the oracle shows ill-conditioned (R19), <= R19_C eps32 round + sens.  Zero failures;
    non-visible particles must have exactly zero gradients.  Returns a summary."""
    vis = status == 0
    V = int(vis.sum())
    n_ent = n_strict = n_ill = n_bad = 0
    worst_cond = 0.0
    fails = []
    for n in G.PARAM_NAMES:
        a, r = gg[n], ref[n]
        assert np.all(a[..., ~vis] == 0.0), (n, "nonzero gradient of a non-visible particle")
        a, r = a[..., vis], r[..., vis]
        s = R19_C * EPS32 * scale["round"][n][..., vis] + scale["sens"][n][..., vis]
        d = np.abs(a - r)
        strict = d <= np.maximum(1e-3 * np.abs(r), 1e-6)
        ok = strict | (d <= s)
        n_ent += d.size
        n_strict += int(strict.sum())
        ill = ok & ~strict
        n_ill += int(ill.sum())
        if ill.any():
            worst_cond = max(worst_cond, float((s[ill] / np.maximum(np.abs(r[ill]), 1e-30)).max()))
        bad = ~ok
        n_bad += int(bad.sum())
        for idx in np.argwhere(bad)[:3]:
            i = tuple(idx)
            fails.append((n, i, float(a[i]), float(r[i]), float(s[i])))
    msg = (f"[grad parity {label}] compared {V} of {V} visible particles ({n_ent} entries): "
           f"{n_strict} within max(1e-3|g|, 1e-6), {n_ill} ill-conditioned (R19, max cond {worst_cond:.3g}) "
           f"within {R19_C:g} eps32 round + sens, {n_bad} failures")
    print(msg)
    assert n_bad == 0, (msg, fails[:10])
    return {"visible": V, "entries": n_ent, "strict": n_strict, "ill_conditioned": n_ill}
