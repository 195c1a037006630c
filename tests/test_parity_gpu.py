"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bars (BASELINE.json north_star):
  * per-particle S1 state, keys, sort order, ranges: bit-exact
  * image: <= 1e-4 max abs per channel, except pixels the oracle flags as
    threshold-ambiguous (R18), which must be rare
  * gradients: |g_gpu - g_ref| <= max(1e-3 |g_ref|, 1e-6), except particles
    touching an ambiguous pixel (reported, bounded in number).
"""
import ctypes as C
import dataclasses

import numpy as np
import pytest
import torch

import ges_inputs as gi
import paper_2402_10128_b200 as G
from paper_2402_10128_b200 import _lib as L
from oracle import oracle as O

from gpu_helpers import (check_grads, gpu_backward, gpu_forward, gpu_keys, masked_upstream, oracle_grads,
                         settings_pair)

pytestmark = pytest.mark.gpu

PRE_KEYS = ("depth", "uv", "conic", "kappa", "rgb", "radius", "rect", "status", "flags")


def compare_preprocess(out, pre):
    P = pre["status"].size
    assert np.array_equal(out["status"], pre["status"])
    c = out["counts"]  # ges_counts: the status census of S1
    assert (c.visible, c.culled_near, c.degenerate, c.offscreen) == tuple(
        int((pre["status"] == k).sum()) for k in (0, 1, 2, 3))
    vis = pre["status"] == 0
    assert np.array_equal(out["depth"].view(np.uint32), pre["depth"].view(np.uint32))
    g_uv = out["pay0"][:, 0:2].T
    g_conic = np.stack([out["pay0"][:, 2], out["pay0"][:, 3], out["pay1"][:, 0]])
    g_kappa = out["pay1"][:, 1]
    g_rgb = np.stack([out["pay1"][:, 2], out["pay1"][:, 3], out["pay2"]])
    for name, g, o in (("uv", g_uv, pre["uv"]), ("conic", g_conic, pre["conic"]), ("kappa", g_kappa, pre["kappa"]),
                       ("rgb", g_rgb, pre["rgb"])):
        gm, om = g[..., vis], o[..., vis]
        bad = np.nonzero(gm.view(np.uint32) != om.view(np.uint32))
        assert bad[0].size == 0, (name, bad[0][:5], gm[bad][:5], om[bad][:5])
    assert np.array_equal(out["radius"][vis], pre["radius"][vis])
    assert np.array_equal(out["rect"].T[:, vis], pre["rect"][:, vis])
    assert np.array_equal(out["flags"][vis], pre["flags"][vis])


def compare_sort(out, pre):
    keys, vals = O.pairs_sorted(pre)
    assert int(out["counts"].pairs) == keys.size
    assert int(out["counts"].slots) == O.count_pairs(pre)
    assert int(out["counts"].visible) == int((pre["status"] == 0).sum())
    assert np.array_equal(out["list"], vals.astype(np.int64))
    assert np.array_equal(gpu_keys(out), keys)
    offsets, _ = O.tile_lists(pre)
    assert np.array_equal(out["ranges"], offsets)


def compare_image(out, ref, tol=1e-4, max_amb_frac=2e-3, alt=None):
    """Image parity: <= tol per channel; at the oracle's flagged pixels (R18) the GPU
    must match the oracle's result or one of its both-branch alternatives (`alt`,
    oracle.render_fwd_alternatives; when given)."""
    amb = ref["amb"] != 0
    assert amb.mean() <= max_amb_frac, amb.mean()
    d = np.abs(out["image"] - ref["image"])
    if alt is not None and amb.any():
        same = (d <= tol).all(axis=0)
        other = np.zeros_like(same)
        for f in range(alt.shape[0]):
            other |= (np.abs(out["image"] - alt[f]) <= tol).all(axis=0)  # (NaN: no such branch)
        bad = amb & ~(same | other)
        print(f"[R18] {int(amb.sum())} flagged pixels: {int((amb & same).sum())} on the oracle's branch, "
              f"{int((amb & ~same & other).sum())} on another, {int(bad.sum())} on neither")
        assert not bad.any(), ("flagged pixels matching neither branch", int(bad.sum()), int(amb.sum()))
    d[:, amb] = 0.0
    assert d.max() <= tol, (d.max(), np.unravel_index(d.argmax(), d.shape))
    ok = ~amb
    assert np.array_equal(out["n_contrib"][ok], ref["n_contrib"][ok])
    assert np.abs(out["final_T"][ok] - ref["final_T"][ok]).max() <= tol
    if "n_eval" in out:
        assert np.array_equal(out["n_eval"][ok], ref["n_eval"][ok])
        assert np.array_equal(out["n_comp"][ok], ref["n_comp"][ok])


def run_case(parts, cam, gs, osx, dL=None, grads=True, max_amb_frac=2e-3, label=""):
    out = gpu_forward(parts, cam, gs)
    assert not out["counts"].overflow
    pre = O.preprocess(parts, cam, osx, "f32")
    compare_preprocess(out, pre)
    compare_sort(out, pre)
    offsets, lst = O.tile_lists(pre)
    ref = O.render_fwd(pre, cam, osx, offsets, lst)
    alt = O.render_fwd_alternatives(pre, cam, osx, offsets, lst, ref["amb"])
    compare_image(out, ref, max_amb_frac=max_amb_frac, alt=alt)
    out["amb_pixels"] = int((ref["amb"] != 0).sum())
    if grads:
        if dL is None:
            dL = gi.upstream_grad(1000, 0, cam.width, cam.height)
        dL = masked_upstream(dL, ref["amb"])
        gg, _ = gpu_backward(out, cam, gs, dL)
        rg, scale = oracle_grads(parts, cam, osx, pre, dL, offsets, lst)
        out["grad_summary"] = check_grads(gg, rg, scale, pre["status"], label)
    return out, pre


def test_config0_full_parity():
    sc = gi.make_config(0)
    gs, osx = settings_pair()
    dL = gi.upstream_grad(sc.seed, 0, 256, 256)
    run_case(sc.particles, sc.cameras[0], gs, osx, dL, label="config 0")


@pytest.mark.parametrize("beta", [0.5, 1.0, 2.0, 4.0, 8.0])
def test_config1_beta_sweep(beta):
    sc = gi.make_config(1, beta_value=beta)
    gs, osx = settings_pair()
    dL = gi.upstream_grad(sc.seed, 0, 512, 512)
    run_case(sc.particles, sc.cameras[0], gs, osx, dL, label=f"config 1 beta={beta}")


# --- the exact GEF kernel of Eq. 2 -----------------
# Its alpha goes through two more MUFU approximations (log2, exp2 of Q^(beta/2)),
# so the oracle's fp32 error bound is wider and flags more threshold-ambiguous
# pixels (R18): up to 1 % of the frame.
EXACT_AMB = 1e-2


def test_exact_kernel_config0_full_parity():
    sc = gi.make_config(0)
    gs, osx = settings_pair(kernel=1)
    run_case(sc.particles, sc.cameras[0], gs, osx, gi.upstream_grad(sc.seed, 0, 256, 256), max_amb_frac=EXACT_AMB,
             label="exact kernel, config 0")


@pytest.mark.parametrize("beta", [0.5, 1.0, 2.0, 4.0, 8.0])
def test_exact_kernel_config1_beta_sweep(beta):
    sc = gi.make_config(1, beta_value=beta, P=20000)
    gs, osx = settings_pair(kernel=1, background=(0.1, 0.2, 0.3))
    run_case(sc.particles, sc.cameras[0], gs, osx, gi.upstream_grad(sc.seed, 0, 512, 512), max_amb_frac=EXACT_AMB,
             label=f"exact kernel, config 1 beta={beta}")


def test_exact_kernel_rejects_nonpositive_beta():
    sc = gi.make_config(0, P=400)
    sc.particles.beta[:7] = np.array([0.0, -1.0, 0.0, -0.5, 0.0, -2.0, 0.0], np.float32)
    gs, osx = settings_pair(kernel=1)
    out, pre = run_case(sc.particles, sc.cameras[0], gs, osx, max_amb_frac=EXACT_AMB)
    assert np.all(out["status"][:7] == O.DEGENERATE)


def test_exact_kernel_frame_mode_must_match():
    sc = gi.make_config(0, P=300)
    cam = sc.cameras[0]
    params = G.PlanarParams.from_inputs(sc.particles)
    r = G.Renderer(params.P, cam.width, cam.height)
    r.forward(params, cam, G.Settings(kernel=1))
    img = torch.empty((3, cam.height, cam.width), dtype=torch.float32, device="cuda")
    with pytest.raises(G.GESError):
        G.ges_render_fwd(r.frame, G.Settings(kernel=0), img)


@pytest.mark.parametrize("mode", [0, 1])
def test_phi_modes_and_background(mode):
    sc = gi.make_config(0, P=1500)
    gs, osx = settings_pair(rho=0.3, phi_mode=mode, background=(0.2, 0.5, 0.9))
    run_case(sc.particles, sc.cameras[0], gs, osx, label=f"phi mode {mode}")


def test_config2_full_view():
    """BASELINE config 2 at full size: 300 K particles, SH 3, one 800x800 view,
    fwd + bwd, every visible particle's gradients compared."""
    sc = gi.make_config(2)
    cam = sc.cameras[2]
    gs, osx = settings_pair()
    run_case(sc.particles, cam, gs, osx, gi.upstream_grad(sc.seed, 2, cam.width, cam.height), label="config 2 view 2")


def test_beta2_bitwise_equals_gaussian_path():
    sc = gi.make_config(1, beta_value=2.0, P=20000)
    cam = sc.cameras[0]
    a = gpu_forward(sc.particles, cam, G.Settings(rho=0.1))
    b = gpu_forward(sc.particles, cam, G.Settings(rho=0.1, gaussian_only=1))
    for k in ("image", "list", "ranges", "pay0", "pay1", "pay2", "final_T", "n_contrib"):
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k


def test_forward_deterministic():
    sc = gi.make_config(0)
    a = gpu_forward(sc.particles, sc.cameras[0], G.Settings())
    b = gpu_forward(sc.particles, sc.cameras[0], G.Settings())
    for k in ("image", "list", "ranges", "final_T", "n_contrib"):
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k


def test_ragged_image_and_tiny_counts():
    # W, H not multiples of 16; P = 1 and P = 37
    for P in (1, 37):
        sc = gi.make_config(0, P=P)
        cam = sc.cameras[0]
        cam = gi.Camera(71, 45, 120.0, 120.0, 35.5, 22.5, 0.2, cam.R, cam.t)
        gs, osx = settings_pair(background=(0.1, 0.1, 0.1))
        run_case(sc.particles, cam, gs, osx, gi.upstream_grad(5, P, 71, 45), label=f"ragged P={P}")


def test_everything_culled():
    sc = gi.make_config(0, P=100)
    parts = sc.particles.subset(slice(None))
    parts.mean[2] = -5.0  # behind the camera
    cam = sc.cameras[0]
    gs, osx = settings_pair(background=(0.3, 0.6, 0.9))
    out = gpu_forward(parts, cam, gs)
    assert out["counts"].visible == 0 and out["counts"].pairs == 0
    bg = np.array([0.3, 0.6, 0.9], np.float32)[:, None, None]
    assert np.array_equal(out["image"], np.broadcast_to(bg, out["image"].shape))
    gg, _ = gpu_backward(out, cam, gs, np.ones((3, 256, 256), np.float32))
    assert all(np.all(v == 0) for v in gg.values())


def test_degenerate_particles():
    sc = gi.make_config(0, P=500)
    parts = sc.particles.subset(slice(None))
    parts.quat[:, :20] = 0.0            # zero quaternion
    parts.log_scale[:, 20:40] = -30.0   # vanishing scale
    parts.log_scale[:, 40:60] = 3.0     # huge: covers the whole screen
    parts.mean[2, 60:80] = 0.2          # exactly on the near plane
    gs, osx = settings_pair()
    run_case(parts, sc.cameras[0], gs, osx, label="degenerate")


def test_overflow_regrow():
    sc = gi.make_config(0)
    cam = sc.cameras[0]
    out = gpu_forward(sc.particles, cam, G.Settings(), pair_capacity=1000)
    c = out["counts"]
    assert not c.overflow and c.capacity >= c.slots > 1000 and c.slots >= c.pairs
    pre = O.preprocess(sc.particles, cam, O.Settings(), "f32")
    compare_sort(out, pre)


def test_gradient_accumulate():
    sc = gi.make_config(0, P=800)
    cam = sc.cameras[0]
    gs, _ = settings_pair()
    out = gpu_forward(sc.particles, cam, gs)
    dL = gi.upstream_grad(3, 0, 256, 256)
    g1, grads = gpu_backward(out, cam, gs, dL)
    g2, _ = gpu_backward(out, cam, gs, dL, accumulate=True, grads=grads)
    for n in G.PARAM_NAMES:
        # float atomics reassociate between the two backward calls: 1e-4 relative, plus
        # a floor of 1e-6 of the group's largest entry for sums that cancel (as in the
        # band test below; a rerun alone moves such entries by ~4e-7 of the maximum)
        floor = 1e-6 + 1e-6 * np.abs(g1[n]).max()
        assert np.all(np.abs(g2[n] - 2 * g1[n]) <= np.maximum(1e-4 * np.abs(g1[n]), floor)), n


def test_full_size_config3_full_frame():
    """BASELINE config 3 at full size (1.5 M particles, 1297x840, SH 3) in the
    launch configuration bench.py times: S1 bit-exact for every particle, every
    key / list / range bit-exact, the whole image, and the gradients of every
    visible particle (fwd + bwd of the full frame)."""
    sc = gi.make_config(3)
    cam = sc.cameras[0]
    gs, osx = settings_pair()
    run_case(sc.particles, cam, gs, osx, gi.upstream_grad(sc.seed, 0, cam.width, cam.height), label="config 3 full frame")


def test_full_size_config4_one_view():
    """BASELINE config 4 at full size (3 M particles, SH 3), one of its 64
    1600x1064 cameras, fwd + bwd, every particle compared."""
    sc = gi.make_config(4, n_views=1)
    cam = sc.cameras[0]
    gs, osx = settings_pair(rho=sc.rho)
    run_case(sc.particles, cam, gs, osx, gi.upstream_grad(sc.seed, 0, cam.width, cam.height), label="config 4 view 0")


@pytest.mark.parametrize("world", [3, 8])
def test_screen_tile_bands_match_full_frame(world):
    """SURVEY.md §8(e) screen-tile bands: band b renders tile rows b, b + N, ...
    Its per-tile lists and its pixels are bit-identical to the full frame's,
    pixels outside the band are untouched, and the S5 gradients of all bands
    sum to the full frame's (atomics reorder the sums: 1e-4 relative)."""
    sc = gi.make_config(2)
    cam = sc.cameras[0]
    gs = G.Settings(rho=sc.rho)
    dL = gi.upstream_grad(sc.seed, 0, cam.width, cam.height)
    out = gpu_forward(sc.particles, cam, gs)
    g_full, _ = gpu_backward(out, cam, gs, dL)
    params = out["params"]
    tx = out["renderer"].frame.c.tiles_x
    ty = out["renderer"].frame.c.tiles_y
    dLt = torch.from_numpy(dL).cuda()
    acc = G.PlanarParams.zeros(params.P, params.sh_degree)
    for b in range(world):
        gb = G.Settings(rho=sc.rho, tile_row_begin=b, tile_row_step=world)
        r = G.Renderer(params.P, cam.width, cam.height)
        img = torch.full((3, cam.height, cam.width), -7.0, device="cuda")
        r.forward(params, cam, gb, image=img)
        r.backward(params, cam, gb, dLt, grads=acc, accumulate=b > 0)
        torch.cuda.synchronize()
        f = r.frame
        rows_t = list(range(b, ty, world))
        assert (f.c.band_begin, f.c.band_step, f.c.band_rows) == (b, world, len(rows_t))
        img = img.cpu().numpy()
        pix = np.zeros(cam.height, bool)
        for t in rows_t:
            pix[16 * t:16 * t + 16] = True
        assert np.array_equal(img[:, pix], out["image"][:, pix])
        assert np.all(img[:, ~pix] == -7.0)
        rng = f.ranges().cpu().numpy().view(np.uint32).astype(np.int64)
        lst = f.list(int(f.counts().pairs)).cpu().numpy().view(np.uint32)
        for k, t in enumerate(rows_t):
            for x in range(tx):
                full = out["list"][out["ranges"][t * tx + x]:out["ranges"][t * tx + x + 1]]
                band = lst[rng[k * tx + x]:rng[k * tx + x + 1]]
                assert np.array_equal(full, band), (b, t, x)
    for n in G.PARAM_NAMES:
        a = getattr(acc, n).cpu().numpy().astype(np.float64)
        # float atomics sum in another order: the north_star gradient tolerance (1e-3
        # relative), plus a floor of 1e-6 of the group's largest entry for sums that cancel
        floor = 1e-6 + 1e-6 * np.abs(g_full[n]).max()
        bad = np.abs(a - g_full[n]) > np.maximum(1e-3 * np.abs(g_full[n]), floor)
        assert bad.sum() == 0, (n, int(bad.sum()))


@pytest.mark.parametrize("case", ["cfg4_camera", "wide_4096", "tall_4096"])
def test_binning_frame_shapes(case):
    """The row and column binnings keep per-lane bin masks for ceil(bins / 32) bins
    per lane (instantiated for 1, 2, 3, 4 and 8): config 4's 1600x1064 camera (100
    tile columns, 67 rows: 4 and 3 per lane), a 4096-wide frame (256 columns: 8 per
    lane) and a 4096-tall frame (256 rows: 8 per lane) must give the same bit-exact
    lists, ranges and images as the oracle."""
    if case == "cfg4_camera":
        sc = gi.make_config(4, P=150000, n_views=1)
        cam = sc.cameras[0]
    else:
        sc = gi.make_config(1, P=40000)
        c0 = sc.cameras[0]
        cam = (gi.Camera(4096, 1024, 900.0, 900.0, 2048.0, 512.0, 0.2, c0.R, c0.t) if case == "wide_4096"
               else gi.Camera(1024, 4096, 900.0, 900.0, 512.0, 2048.0, 0.2, c0.R, c0.t))
    gs, osx = settings_pair(rho=sc.rho)
    run_case(sc.particles, cam, gs, osx, gi.upstream_grad(sc.seed, 4, cam.width, cam.height), label=case)


def test_binning_stage_overflow_writes_directly():
    """A chunk whose row-list entries (rows) or pairs (columns) exceed its shared-memory
    stage writes them straight to HBM instead of staging them (bin.cu).  Wide splats
    (rects of ~20-40 tiles a side) push every chunk over its stage: S1 state, lists and
    ranges bit-exact against the oracle, and the image within the north_star bar."""
    sc = gi.random_small_scene(23, P=5000, W=1024, H=768, sh_degree=1, kappa_max=0.6, log_scale_mu=-0.8)
    cam = sc.cameras[0]
    gs, osx = settings_pair(rho=sc.rho)
    out = gpu_forward(sc.particles, cam, gs)
    pre = O.preprocess(sc.particles, cam, osx, "f32")
    compare_preprocess(out, pre)
    compare_sort(out, pre)
    vis = pre["status"] == 0
    h = (pre["rect"][3] - pre["rect"][1])[vis]
    w = (pre["rect"][2] - pre["rect"][0])[vis]
    assert np.median(h) * 2048 > 8192 and np.median(w) * 3072 > 16384  # every chunk overflows its stage
    ref = O.render_fwd(pre, cam, osx, *O.tile_lists(pre))
    compare_image(out, ref)


def test_exact_kernel_bands_match_full_frame():
    """Screen-tile bands with the exact GEF kernel: every band's
    pixels bit-identical to the full frame's, and the bands' S5 gradients sum to the
    full frame's (float atomics reorder: the tolerance of the Gaussian band test)."""
    sc = gi.make_config(1, P=20000)
    cam = sc.cameras[0]
    gs = G.Settings(rho=sc.rho, kernel=1)
    dL = gi.upstream_grad(sc.seed, 0, cam.width, cam.height)
    out = gpu_forward(sc.particles, cam, gs)
    g_full, _ = gpu_backward(out, cam, gs, dL)
    params = out["params"]
    dLt = torch.from_numpy(dL).cuda()
    acc = G.PlanarParams.zeros(params.P, params.sh_degree)
    world = 3
    for b in range(world):
        gb = G.Settings(rho=sc.rho, kernel=1, tile_row_begin=b, tile_row_step=world)
        r = G.Renderer(params.P, cam.width, cam.height)
        img = torch.full((3, cam.height, cam.width), -7.0, device="cuda")
        r.forward(params, cam, gb, image=img)
        r.backward(params, cam, gb, dLt, grads=acc, accumulate=b > 0)
        torch.cuda.synchronize()
        img = img.cpu().numpy()
        pix = np.zeros(cam.height, bool)
        for t in range(b, r.frame.c.tiles_y, world):
            pix[16 * t:16 * t + 16] = True
        assert np.array_equal(img[:, pix], out["image"][:, pix])
        assert np.all(img[:, ~pix] == -7.0)
    for n in G.PARAM_NAMES:
        a = getattr(acc, n).cpu().numpy().astype(np.float64)
        floor = 1e-6 + 1e-6 * np.abs(g_full[n]).max()
        bad = np.abs(a - g_full[n]) > np.maximum(1e-3 * np.abs(g_full[n]), floor)
        assert bad.sum() == 0, (n, int(bad.sum()))


def test_step_captured_as_cuda_graph_matches_direct_launches():
    """The API is stream-ordered and capture-safe (bench.py replays S1-S5 as one CUDA
    graph): a captured step reproduces the directly launched step's image and lists
    bit for bit, and its gradients up to float-atomic reordering."""
    sc = gi.make_config(1, P=20000)
    cam = sc.cameras[0]
    st = G.Settings(rho=sc.rho)
    params = G.PlanarParams.from_inputs(sc.particles)
    r = G.Renderer(params.P, cam.width, cam.height)
    img0 = torch.empty((3, cam.height, cam.width), device="cuda")
    r.forward(params, cam, st, image=img0)
    r.grow(int(r.frame.counts().slots))
    frame = r.frame
    dL = torch.from_numpy(gi.upstream_grad(sc.seed, 0, cam.width, cam.height)).cuda()
    s = torch.cuda.current_stream()
    img_a = torch.empty_like(img0)
    g_a = G.PlanarParams.zeros(params.P, params.sh_degree)
    G.ges_preprocess(params, cam, st, frame, s)
    G.ges_sort(frame, s)
    G.ges_render_fwd(frame, st, img_a, None, s)
    G.ges_render_bwd(params, cam, st, frame, dL, g_a, False, s)
    torch.cuda.synchronize()
    lst_a = frame.list(int(frame.counts().pairs)).clone()
    img_b = torch.full_like(img0, -1.0)
    g_b = G.PlanarParams.zeros(params.P, params.sh_degree)
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(s)
    with torch.cuda.graph(graph, stream=cap):
        G.ges_preprocess(params, cam, st, frame, cap)
        G.ges_sort(frame, cap)
        G.ges_render_fwd(frame, st, img_b, None, cap)
        G.ges_render_bwd(params, cam, st, frame, dL, g_b, False, cap)
    s.wait_stream(cap)
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(img_a, img_b)
    assert torch.equal(lst_a, frame.list(int(frame.counts().pairs)))
    a, b = g_a.flat.cpu().numpy(), g_b.flat.cpu().numpy()
    floor = 1e-6 + 1e-6 * np.abs(a).max()
    assert np.all(np.abs(a - b) <= np.maximum(1e-4 * np.abs(a), floor))


@pytest.mark.parametrize("P", [2000, 60000])
def test_equal_depth_ties_keep_index_order(P):
    """R11: equal depth keys are ordered by particle index.  Every particle at the
    same camera depth (z = 4 exactly) spread over the image: the single-sweep depth
    sort must be stable across warps, tiles and CTAs (60 K particles: several CTAs),
    so every tile's list is in index order; S1 state, lists, image and gradients
    against the oracle."""
    sc = gi.make_config(1, beta_value=2.0, P=P)
    parts = sc.particles.subset(slice(None))
    parts.mean[2] = 4.0
    cam = sc.cameras[0]
    gs, osx = settings_pair()
    out, pre = run_case(parts, cam, gs, osx, gi.upstream_grad(sc.seed, 0, cam.width, cam.height),
                        label=f"equal depths P={P}")
    r = out["ranges"]
    for t in range(r.size - 1):
        seg = out["list"][r[t]:r[t + 1]]
        assert np.all(np.diff(seg) > 0), t


def test_band_without_rows():
    """A band that owns no tile row (N bands > tile rows, band b >= tiles_y) renders
    nothing: every stage runs (no zero-size launch), no pairs, the image is untouched
    and the gradients are zero."""
    sc = gi.make_config(0)
    cam = sc.cameras[0]
    assert (cam.height + 15) // 16 == 16
    gs = G.Settings(rho=0.1, tile_row_begin=17, tile_row_step=20)
    params = G.PlanarParams.from_inputs(sc.particles)
    r = G.Renderer(params.P, cam.width, cam.height)
    img = torch.full((3, cam.height, cam.width), 7.0, device="cuda")
    G.ges_preprocess(params, cam, gs, r.frame)
    G.ges_sort(r.frame)
    G.ges_render_fwd(r.frame, gs, img)
    dL = torch.from_numpy(gi.upstream_grad(1, 0, cam.width, cam.height)).cuda()
    grads = G.PlanarParams.zeros(params.P, params.sh_degree)
    grads.flat.fill_(5.0)
    G.ges_render_bwd(params, cam, gs, r.frame, dL, grads)
    torch.cuda.synchronize()
    c = r.frame.counts()
    assert c.visible == 0 and c.pairs == 0 and not c.overflow
    assert r.frame.c.band_rows == 0
    assert bool((img == 7.0).all())
    assert bool((grads.flat == 0.0).all())


@pytest.mark.parametrize("case", ["config0", "config1_beta2", "config0_exact"])
def test_mean2d_gradient(case):
    """ges_grads.mean2d (optional output): dL/d(u, v), the gradient of each visible
    particle's projected mean in pixels, against the oracle's S5a du, dv (Eq. 3's
    adjoint) at the north_star tolerance or the entry's R19 scale; exactly 0 for
    particles that are not visible; accumulate adds."""
    kernel = 1 if case.endswith("exact") else 0
    sc = gi.make_config(1, beta_value=2.0, P=20000) if case == "config1_beta2" else gi.make_config(0)
    cam = sc.cameras[0]
    gs, osx = settings_pair(rho=0.1, kernel=kernel)
    out = gpu_forward(sc.particles, cam, gs)
    pre = O.preprocess(sc.particles, cam, osx, "f32")
    offsets, lst = O.tile_lists(pre)
    ref = O.render_fwd(pre, cam, osx, offsets, lst)
    dL = masked_upstream(gi.upstream_grad(sc.seed, 3, cam.width, cam.height), ref["amb"])
    g2d, mag = O.render_bwd(pre, cam, osx, offsets, lst, dL, with_abs=True)
    P = sc.particles.P
    m2d = torch.full((2, P), 3.0, device="cuda")
    grads = G.PlanarParams.zeros(P, out["params"].sh_degree)
    dLt = torch.from_numpy(np.ascontiguousarray(dL, np.float32)).cuda()
    G.ges_render_bwd(out["params"], cam, gs, out["renderer"].frame, dLt, grads, mean2d=m2d)
    torch.cuda.synchronize()
    a = m2d.cpu().numpy().astype(np.float64)
    vis = pre["status"] == 0
    assert np.all(a[:, ~vis] == 0.0)
    from gpu_helpers import EPS32, R19_C
    for j in range(2):
        r = g2d[j, vis]
        bound = np.maximum(np.maximum(1e-3 * np.abs(r), 1e-6), R19_C * EPS32 * mag[j, vis] + mag[10 + j, vis])
        bad = np.abs(a[j, vis] - r) > bound
        assert bad.sum() == 0, (case, j, int(bad.sum()), int(vis.sum()))
    print(f"[mean2d {case}] compared {int(vis.sum())} of {int(vis.sum())} visible particles")
    # accumulate: a second view adds
    G.ges_preprocess(out["params"], cam, gs, out["renderer"].frame)
    G.ges_sort(out["renderer"].frame)
    G.ges_render_fwd(out["renderer"].frame, gs, torch.empty(3, cam.height, cam.width, device="cuda"))
    G.ges_render_bwd(out["params"], cam, gs, out["renderer"].frame, dLt, grads, accumulate=True, mean2d=m2d)
    torch.cuda.synchronize()
    b = m2d.cpu().numpy().astype(np.float64)
    assert np.allclose(b, 2 * a, rtol=1e-4, atol=1e-6 * (1 + np.abs(a).max()))


def test_count_nonfinite():
    """Failure detection (ges_count_nonfinite): counts NaN and +-Inf exactly, 0 on a
    rendered frame and its gradients; accumulates over several buffers."""
    x = torch.randn(1000003, device="cuda")
    assert int(G.count_nonfinite(x).item()) == 0
    x[[0, 17, 999999]] = float("nan")
    x[[5, 1000002]] = float("inf")
    x[123] = -float("inf")
    assert int(G.count_nonfinite(x).item()) == 6
    assert int(G.count_nonfinite(x, x[:10].contiguous()).item()) == 8
    sc = gi.make_config(0)
    out = gpu_forward(sc.particles, sc.cameras[0], G.Settings())
    _, grads = gpu_backward(out, sc.cameras[0], G.Settings(), gi.upstream_grad(1, 0, 256, 256))
    img = torch.from_numpy(out["image"]).cuda()
    assert int(G.count_nonfinite(img, grads.flat).item()) == 0


def test_sh_grad_from_colour_matches_accumulated_sh():
    """SH-factorised view exchange: the SH gradient rebuilt from the
    per-view dL/drgb (ges_grads.drgb) and the cameras by ges_sh_grad_from_colour equals
    the SH planes S5b accumulates over the same views (same per-view products, the sum
    order may differ by one rounding: rtol 1e-5 of the summed magnitudes).  A single
    view in overwrite mode agrees to the same bound; invalid arguments are rejected."""
    sc = gi.make_config(2, P=30000, n_views=4)
    gs = G.Settings()
    dev = G.PlanarParams.from_inputs(sc.particles)
    P, V = dev.P, len(sc.cameras)
    r = G.Renderer(P, sc.cameras[0].width, sc.cameras[0].height)
    grads = G.PlanarParams.zeros(P, dev.sh_degree)
    drgb = torch.zeros((V, 3, P), device="cuda")
    one_sh = []
    for v, cam in enumerate(sc.cameras):
        r.forward(dev, cam, gs)
        dL = torch.from_numpy(np.ascontiguousarray(gi.upstream_grad(sc.seed, v, cam.width, cam.height),
                                                   np.float32)).cuda()
        G.ges_render_bwd(dev, cam, gs, r.frame, dL, grads, accumulate=v > 0, drgb=drgb[v])
        if v == 0:
            one_sh.append(grads.sh.clone())
    cams = G.camera_rows(sc.cameras)
    torch.cuda.synchronize()
    assert int((drgb.abs().sum(dim=1) > 0).sum().item()) > 0.1 * P * V
    rebuilt = G.sh_grad_from_colour(dev, cams, drgb)
    torch.cuda.synchronize()
    # magnitude of the sum's terms: |Y_k| <= 1.1 at degree 3 -> bound by sum_v |drgb_v|
    mag = drgb.abs().sum(dim=0).repeat(dev.sh.shape[0] // 3, 1)
    assert torch.all((rebuilt - grads.sh).abs() <= 1e-5 * mag + 1e-12), float((rebuilt - grads.sh).abs().max())
    one = G.sh_grad_from_colour(dev, cams[:1].contiguous(), drgb[:1].contiguous())
    torch.cuda.synchronize()
    assert torch.all((one - one_sh[0]).abs() <= 1e-6 * mag + 1e-12)
    # accumulate adds; zero views leave an overwrite at 0
    acc = rebuilt.clone()
    G.sh_grad_from_colour(dev, cams, drgb, out=acc, accumulate=True)
    assert torch.allclose(acc, 2 * rebuilt, rtol=1e-6, atol=0)
    z = G.sh_grad_from_colour(dev, cams[:0].contiguous(), drgb[:0].contiguous())
    assert int((z != 0).sum().item()) == 0
    lib = L.load()
    st = lib.ges_sh_grad_from_colour(C.c_void_p(dev.mean.data_ptr()), P, 4, C.c_void_p(cams.data_ptr()), V,
                                     C.c_void_p(drgb.data_ptr()), C.c_void_p(rebuilt.data_ptr()), 0, None)
    assert st == L.GES_ERR_INVALID_ARG
    st = lib.ges_sh_grad_from_colour(C.c_void_p(dev.mean.data_ptr()), P, 3, None, V,
                                     C.c_void_p(drgb.data_ptr()), C.c_void_p(rebuilt.data_ptr()), 0, None)
    assert st == L.GES_ERR_INVALID_ARG


def test_backward_launch_order():
    """ges_frame.tile_order (S4 -> S5a launch order): after one forward the 64 buckets hold
    every tile exactly once, in the bucket of the tile's largest n_contrib; S5a's gradients
    equal those of the index-order fallback (a second S4 on the same frame doubles the
    bucket counts) up to float-atomic order; band frames too."""
    sc = gi.make_config(2, P=60000, n_views=1)
    cam = sc.cameras[0]
    gs = G.Settings(rho=sc.rho)
    dev = G.PlanarParams.from_inputs(sc.particles)
    dL = torch.from_numpy(np.ascontiguousarray(gi.upstream_grad(sc.seed, 0, cam.width, cam.height))).cuda()
    for band in ((0, 1), (1, 3)):
        s = dataclasses.replace(gs, tile_row_begin=band[0], tile_row_step=band[1])
        r = G.Renderer(dev.P, cam.width, cam.height)
        img = r.forward(dev, cam, s)
        f = r.frame
        T = f.c.tiles_x * f.c.band_rows
        torch.cuda.synchronize()
        counts = f.view("tile_bucket", torch.int32, 64).cpu().numpy()
        assert counts.sum() == T
        order = f.view("tile_order", torch.int32, 64 * T).cpu().numpy().reshape(64, T)
        tiles = np.concatenate([order[b, :counts[b]] for b in range(64)])
        assert np.array_equal(np.sort(tiles), np.arange(T))
        # bucket = the 4-per-octave log bucket of the tile's largest n_contrib
        H, W = cam.height, cam.width
        nc = f.view("n_contrib", torch.int32, W * H).cpu().numpy().reshape(H, W).astype(np.int64)
        rows = [band[0] + k * band[1] for k in range(f.c.band_rows)]
        for b in range(64):
            for t in order[b, :counts[b]]:
                ty, tx = rows[t // f.c.tiles_x], t % f.c.tiles_x
                c = int(nc[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16].max())
                e = c.bit_length() - 1
                want = c if c < 4 else min(63, 4 * (e - 1) + ((c >> (e - 2)) & 3))
                assert b == want, (t, c, b, want)
        g1 = r.backward(dev, cam, s, dL).flat.clone()
        G.ges_render_fwd(f, s, img)               # second S4: counts 2T -> index order
        torch.cuda.synchronize()
        assert f.view("tile_bucket", torch.int32, 64).cpu().numpy().sum() == 2 * T
        g2 = r.backward(dev, cam, s, dL).flat.clone()
        torch.cuda.synchronize()
        a, b2 = g1.cpu().numpy(), g2.cpu().numpy()
        assert np.all(np.abs(a - b2) <= 1e-4 * np.abs(a) + 1e-6 * (1 + np.abs(a).max()))


@pytest.mark.parametrize("case", ["config0", "config1_beta2", "config0_clamped"])
def test_drgb_output_parity(case):
    """ges_grads.drgb (optional output, the per-view colour gradient of the SH-factorised
    exchange): dL/d rgb of every visible particle against the oracle's S5a colour sums
    (g2d rows 6-8) with the clamped channels zeroed (flags bits 0-2, R13), at the
    north_star tolerance or the entry's R19 scale; exactly 0 for particles that are not
    visible."""
    sc = gi.make_config(1, beta_value=2.0, P=20000) if case == "config1_beta2" else gi.make_config(0)
    parts = sc.particles
    if case.endswith("clamped"):  # a third of the particles with one or two channels below 0
        parts = parts.subset(slice(None))
        parts.sh[0, 0::3] = -3.0
        parts.sh[2, 0::6] = -3.0
    cam = sc.cameras[0]
    gs, osx = settings_pair(rho=0.1)
    out = gpu_forward(parts, cam, gs)
    pre = O.preprocess(parts, cam, osx, "f32")
    offsets, lst = O.tile_lists(pre)
    ref = O.render_fwd(pre, cam, osx, offsets, lst)
    dL = masked_upstream(gi.upstream_grad(sc.seed, 5, cam.width, cam.height), ref["amb"])
    g2d, mag = O.render_bwd(pre, cam, osx, offsets, lst, dL, with_abs=True)
    P = parts.P
    drgb = torch.full((3, P), 7.0, device="cuda")
    grads = G.PlanarParams.zeros(P, out["params"].sh_degree)
    dLt = torch.from_numpy(np.ascontiguousarray(dL, np.float32)).cuda()
    G.ges_render_bwd(out["params"], cam, gs, out["renderer"].frame, dLt, grads, drgb=drgb)
    torch.cuda.synchronize()
    a = drgb.cpu().numpy().astype(np.float64)
    vis = pre["status"] == 0
    assert np.all(a[:, ~vis] == 0.0)
    from gpu_helpers import EPS32, R19_C
    n_clamped = 0
    for ch in range(3):
        clamped = (pre["flags"][vis] >> ch) & 1 == 1
        n_clamped += int(clamped.sum())
        r = np.where(clamped, 0.0, g2d[6 + ch, vis])
        bound = np.maximum(np.maximum(1e-3 * np.abs(r), 1e-6),
                           R19_C * EPS32 * mag[6 + ch, vis] + mag[16 + ch, vis])
        bad = np.abs(a[ch, vis] - r) > bound
        assert bad.sum() == 0, (case, ch, int(bad.sum()), int(vis.sum()))
        assert np.all(a[ch, vis][clamped] == 0.0)
    print(f"[drgb {case}] compared {int(vis.sum())} of {int(vis.sum())} visible particles, "
          f"{n_clamped} clamped channels")
    if case.endswith("clamped"):
        assert n_clamped > 100


def test_sh_grad_from_colour_against_oracle():
    """ges_sh_grad_from_colour over several views against the oracle: the sum over the
    views of the oracle's S5b SH gradient of each view (oracle S5a -> S5b, fp64), the
    GPU side fed with the views' dL/drgb from ges_grads.drgb.  Tolerance: 1e-3 of the
    summed magnitudes of the views' terms (grad_magnitude) + 1e-6."""
    sc = gi.make_config(2, P=20000, n_views=3)
    parts = sc.particles
    gs, osx = settings_pair(rho=sc.rho)
    dev = G.PlanarParams.from_inputs(parts)
    P, V = dev.P, len(sc.cameras)
    cam0 = sc.cameras[0]
    r = G.Renderer(P, cam0.width, cam0.height)
    grads = G.PlanarParams.zeros(P, dev.sh_degree)
    drgb = torch.zeros((V, 3, P), device="cuda")
    want = np.zeros((3 * parts.K, P))
    mag = np.zeros((3 * parts.K, P))
    for v, cam in enumerate(sc.cameras):
        pre = O.preprocess(parts, cam, osx, "f32")
        offsets, lst = O.tile_lists(pre)
        ref = O.render_fwd(pre, cam, osx, offsets, lst)
        dL = masked_upstream(gi.upstream_grad(sc.seed, v, cam.width, cam.height), ref["amb"])
        g2d, gabs = O.render_bwd(pre, cam, osx, offsets, lst, dL, with_abs=True)
        want += O.backward_particles(parts, cam, osx, g2d, pre["status"], pre["flags"])["sh"]
        mag += O.grad_magnitude(parts, cam, osx, gabs, pre["status"], pre["flags"])["sh"]
        r.forward(dev, cam, gs)
        dLt = torch.from_numpy(np.ascontiguousarray(dL, np.float32)).cuda()
        G.ges_render_bwd(dev, cam, gs, r.frame, dLt, grads, drgb=drgb[v])
    got = G.sh_grad_from_colour(dev, G.camera_rows(sc.cameras), drgb).cpu().numpy().astype(np.float64)
    bad = np.abs(got - want) > 1e-3 * mag + 1e-6
    assert bad.sum() == 0, (int(bad.sum()), float(np.abs(got - want).max()))
    nz = int((np.abs(want) > 0).any(axis=0).sum())
    assert nz > 0.2 * P
    print(f"[sh from colour] {V} views, {nz} particles with an SH gradient, all {3 * parts.K * P} entries compared")
