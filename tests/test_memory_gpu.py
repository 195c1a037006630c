"""Memory safety and determinism of the CUDA path without compute-sanitizer (closed on this
GPU pool): own checks in its place.

* uninitialized reads (initcheck's job): the frame workspace is POISONED (every byte 0xA5,
  except frame.grad2d, which ges.h requires zeroed) instead of zero-filled; every output
  must be bit-identical to a run on a zeroed workspace (forward, lists) and the gradients
  must pass the oracle parity check.
* out-of-bounds writes (memcheck's job): guard bands around every output buffer (image,
  gradients) and after the workspace, plus the alignment padding between the frame's
  sub-arrays (ges_frame_layout), all poisoned; not one byte may change.
* races (racecheck's job, in part): the forward and the lists are bit-identical run to run;
  the backward's float-atomic sums are compared run to run with a max-ulp report.
Cases: configs 0 and 1, the exact-beta kernel, screen-tile bands, a ragged tiny frame.
"""
import numpy as np
import pytest
import torch

import ges_inputs as gi
import paper_2402_10128_b200 as G
from oracle import oracle as O

from gpu_helpers import check_grads, masked_upstream, oracle_grads

pytestmark = pytest.mark.gpu

POISON = 0xA5
GUARD = 4096  # bytes


def _guarded(n_floats, device="cuda"):
    """A float32 view of n_floats inside a poisoned buffer with GUARD bytes on both sides."""
    g = GUARD // 4
    buf = torch.full((n_floats + 2 * g,), 0, dtype=torch.int32, device=device)
    buf.fill_(int(np.int32(np.uint32(0xA5A5A5A5))))
    return buf, buf[g:g + n_floats].view(torch.float32)


def _guards_intact(buf, n_floats):
    g = GUARD // 4
    pat = int(np.int32(np.uint32(0xA5A5A5A5)))
    return bool((buf[:g] == pat).all()) and bool((buf[g + n_floats:] == pat).all())


def _run(parts, cam, st, poison):
    P, W, H = parts.P, cam.width, cam.height
    params = G.PlanarParams.from_inputs(parts)
    r0 = G.Renderer(P, W, H)
    r0.forward(params, cam, st)
    cap = int(r0.frame.counts().slots * 1.25) + 64
    frame = G.Frame(P, W, H, cap, poison=poison, guard=GUARD)
    ibuf, img = _guarded(3 * W * H)
    img = img.view(3, H, W)
    C = params.flat.shape[0]
    gbuf, gflat = _guarded(C * P)
    grads = G.PlanarParams(gflat.view(C, P), P, params.sh_degree)
    dL = gi.upstream_grad(7, 0, W, H)
    G.ges_preprocess(params, cam, st, frame)
    G.ges_sort(frame)
    G.ges_render_fwd(frame, st, img)
    torch.cuda.synchronize()
    assert not frame.counts().overflow
    return params, frame, ibuf, img, gbuf, grads, dL


def _padding_intact(frame):
    """Bytes between the frame's sub-arrays (and after the workspace) still hold the poison."""
    lay = sorted(frame.layout().items(), key=lambda kv: kv[1][0])
    ws = frame.ws[frame.offset:].cpu().numpy()
    zero_end = frame.c.zero_bytes
    bad = []
    for (name, (o, s)), (_, (o2, _)) in zip(lay, lay[1:] + [("end", (frame.nbytes, 0))]):
        pad = ws[o + s:o2]
        if o + s >= zero_end and pad.size and not np.all(pad == POISON):
            bad.append((name, int(np.count_nonzero(pad != POISON)), pad.size))
    tail = ws[frame.nbytes:]
    if not np.all(tail == POISON):
        bad.append(("tail guard", int(np.count_nonzero(tail != POISON)), tail.size))
    return bad


CASES = {
    "config0": lambda: (gi.make_config(0).particles, gi.make_config(0).cameras[0], G.Settings(rho=0.1),
                        O.Settings(rho=0.1)),
    "config0_exact": lambda: (gi.make_config(0).particles, gi.make_config(0).cameras[0], G.Settings(rho=0.1, kernel=1),
                              O.Settings(rho=0.1, kernel=1)),
    "config1_beta2": lambda: (gi.make_config(1, beta_value=2.0, P=20000).particles,
                              gi.make_config(1, beta_value=2.0, P=20000).cameras[0], G.Settings(rho=0.1),
                              O.Settings(rho=0.1)),
    "band_1_of_3": lambda: (gi.make_config(0).particles, gi.make_config(0).cameras[0],
                            G.Settings(rho=0.1, tile_row_begin=1, tile_row_step=3), None),
    "ragged_tiny": lambda: (gi.make_config(0, P=37).particles,
                            gi.Camera(71, 45, 120.0, 120.0, 35.5, 22.5, 0.2, np.eye(3, dtype=np.float32),
                                      np.zeros(3, np.float32)),
                            G.Settings(rho=0.1, background=(0.1, 0.1, 0.1)), O.Settings(rho=0.1,
                                                                                      background=(0.1, 0.1, 0.1))),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_poisoned_workspace_and_guard_bands(case):
    parts, cam, gst, ost = CASES[case]()
    p1, f1, ib1, img1, gb1, gr1, dL = _run(parts, cam, gst, POISON)
    p0, f0, ib0, img0, gb0, gr0, _ = _run(parts, cam, gst, None)
    # forward: bit-identical to the zero-filled workspace
    assert torch.equal(img1.view(torch.int32), img0.view(torch.int32)), "image depends on workspace contents"
    M = int(f1.counts().pairs)
    assert M == int(f0.counts().pairs)
    T = f1.c.band_rows * f1.c.tiles_x   # (a band frame's ranges cover its own tile rows only)
    assert torch.equal(f1.list(M), f0.list(M)) and torch.equal(f1.ranges()[:T + 1], f0.ranges()[:T + 1])
    # backward on the poisoned frame
    if ost is not None:
        ref = O.render_fwd(O.preprocess(parts, cam, ost, "f32"), cam, ost,
                           *O.tile_lists(O.preprocess(parts, cam, ost, "f32")))
        dL = masked_upstream(dL, ref["amb"])
    dLt = torch.from_numpy(np.ascontiguousarray(dL)).cuda()
    G.ges_render_bwd(p1, cam, gst, f1, dLt, gr1)
    torch.cuda.synchronize()
    assert _guards_intact(ib1, 3 * cam.width * cam.height), "write outside the image"
    assert _guards_intact(gb1, gr1.flat.numel()), "write outside the gradient buffer"
    bad = _padding_intact(f1)
    assert not bad, f"writes into the frame's padding / tail guard: {bad}"
    if ost is not None:
        pre = O.preprocess(parts, cam, ost, "f32")
        rg, scale = oracle_grads(parts, cam, ost, pre, dL)
        gg = {n: getattr(gr1, n).cpu().numpy().astype(np.float64) for n in G.PARAM_NAMES}
        check_grads(gg, rg, scale, pre["status"], f"poisoned workspace, {case}")
    else:
        assert torch.isfinite(gr1.flat).all()


def _ulps(a, b):
    """|a - b| in units of the last place of max(|a|, |b|) (fp32)."""
    m = np.maximum(np.abs(a), np.abs(b)).astype(np.float32)
    ulp = np.spacing(np.maximum(m, np.float32(1e-30))).astype(np.float64)
    return np.abs(a.astype(np.float64) - b.astype(np.float64)) / ulp


@pytest.mark.parametrize("cfg", [0, 1])
def test_backward_determinism_max_ulp(cfg):
    """Run-to-run: the forward (image, lists, final T, n_contrib) is bit-identical; the
    backward differs only by the reassociation of its float-atomic sums.  Reports the
    max difference in ulps per parameter group, and bounds every entry by the R19 scale
    of the oracle (the reassociation of the same fp32 terms)."""
    sc = gi.make_config(cfg, **({"beta_value": 2.0, "P": 20000} if cfg == 1 else {}))
    cam = sc.cameras[0]
    st = G.Settings(rho=0.1)
    params = G.PlanarParams.from_inputs(sc.particles)
    r = G.Renderer(params.P, cam.width, cam.height)
    dL = torch.from_numpy(gi.upstream_grad(sc.seed, 0, cam.width, cam.height)).cuda()
    outs = []
    for _ in range(3):
        img = r.forward(params, cam, st).clone()
        M = int(r.frame.counts().pairs)
        lst = r.frame.list(M).clone()
        fT = r.frame.view("final_T", torch.float32, cam.width * cam.height).clone()
        g = r.backward(params, cam, st, dL)
        torch.cuda.synchronize()
        outs.append((img, lst, fT, g.flat.cpu().numpy().copy()))
    for img, lst, fT, _ in outs[1:]:
        assert torch.equal(img, outs[0][0]) and torch.equal(lst, outs[0][1]) and torch.equal(fT, outs[0][2])
    pre = O.preprocess(sc.particles, cam, O.Settings(rho=0.1), "f32")
    _, scale = oracle_grads(sc.particles, cam, O.Settings(rho=0.1), pre, dL.cpu().numpy())
    from gpu_helpers import EPS32, R19_C
    bound = np.concatenate([
        np.atleast_2d(R19_C * EPS32 * scale["round"][n] + scale["sens"][n]) for n in G.PARAM_NAMES], axis=0)
    report = []
    for k in range(1, len(outs)):
        a, b = outs[0][3], outs[k][3]
        u = _ulps(a, b)
        report.append(float(u.max()))
        assert np.all(np.abs(a.astype(np.float64) - b) <= bound + 1e-30)
    print(f"[determinism config {cfg}] forward bit-identical over {len(outs)} runs; backward max ulp diff "
          f"{max(report):.0f} (median over entries {float(np.median(_ulps(outs[0][3], outs[1][3]))):.1f})")


def test_sort_protocols_repeatable_under_load():
    """The sort's and binning's cross-CTA protocols (chunk tickets, published words,
    two-level look-backs) give the same lists and ranges frame after frame: 200
    back-to-back frames of config 3 (10 compared bit for bit with the first)."""
    sc = gi.make_config(3)
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
    for it in range(200):
        G.ges_preprocess(params, cam, st, r.frame)
        G.ges_sort(r.frame)
        if it % 20 == 19:
            torch.cuda.synchronize()
            assert int(r.frame.counts().pairs) == M
            assert torch.equal(r.frame.list(M), ref_list) and torch.equal(r.frame.ranges(), ref_rng), it
