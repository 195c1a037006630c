"""Pins of the CPU oracle against what the paper and mathematics fix (not the
oracle's own formulas).  Runs on CPU (`-m "not gpu"`).

Each test names the passage it pins.  A plausible mistake anywhere in the
oracle (a dropped term, a wrong sign, a transposed operand) fails one of them:
  * exp_spec                  vs libm exp in fp64 (<= 2 ulp), exp(0) = 1
  * log_spec                  vs libm log in fp64 (<= 3 ulp), log(2^k) = k ln2
  * tile rect (R10)           brute-force alpha over every pixel; the 'all'
                              membership (every particle in every tile) gives
                              the same image and gradients
  * phi-bar, Eq. 6            golden values from tests/golden/phi_bar.txt
  * Sigma, S*phi, EWA         vs scipy rotation + numerically differentiated
                              pinhole projection (independent Jacobian)
  * kernel value              one isotropic particle on the optical axis:
                              textbook Gaussian at sample pixels, all beta
  * Eq. 3 compositing         T + sum(w) = 1, empty scene, single splat,
                              permutation invariance, convexity
  * keys / lists              numpy brute force on tiny inputs
  * adjoints                  central finite differences of the all-fp64
                              pipeline, every parameter group incl. beta
  * beta chain identity       dL/dbeta = rho (1 - phi/2) sum_k dL/dlog s_k
  * beta = 2 / rho = 0        bit-identical to the Gaussian path (Fig. 4)
  * SH basis                  orthonormality by Gauss-Legendre quadrature
"""
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import ges_inputs as gi
from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden_phi():
    rows = []
    with open(os.path.join(GOLDEN, "phi_bar.txt")) as f:
        for line in f:
            if line.startswith("#") or line.startswith("gamma"):
                continue
            b, r, v = line.split()
            rows.append((float(b), float(r), float(v)))
    return rows


def one_particle(mean, log_scale, quat=(1, 0, 0, 0), logit=0.0, beta=2.0, sh=None, sh_degree=0):
    K = (sh_degree + 1) ** 2
    if sh is None:
        sh = np.zeros((3 * K, 1))
        sh[0:3, 0] = 0.5
    f = lambda a: np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, 1), np.float32)
    return gi.Particles(f(mean), f(log_scale), f(quat), np.array([logit], np.float32),
                        np.ascontiguousarray(sh, np.float32), np.array([beta], np.float32), sh_degree)


def cam_identity(W=64, H=64, f=60.0, near=0.2):
    return gi.Camera(W, H, f, f, W / 2.0, H / 2.0, near, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))


# --------------------------------------------------------------------------
# KEYSPEC exp
# --------------------------------------------------------------------------
def test_exp_spec_accuracy_and_exact_zero():
    x = np.linspace(-87.0, 88.0, 400001, dtype=np.float32)
    y = O.exp_spec(x).astype(np.float64)
    ref = np.exp(x.astype(np.float64))
    ulp = np.spacing(ref.astype(np.float32)).astype(np.float64)
    err = np.abs(y - ref) / ulp
    assert err.max() <= 2.0, err.max()
    assert O.exp_spec(np.array([0.0], np.float32))[0] == np.float32(1.0)
    # reproducible bit pattern (no hidden state)
    assert np.array_equal(O.exp_spec(x).view(np.uint32), O.exp_spec(x).view(np.uint32))


# --------------------------------------------------------------------------
# phi-bar (Eq. 6) through the whole S1: one isotropic particle on the axis
# --------------------------------------------------------------------------
@pytest.mark.parametrize("mode", [O.PHI_SCALE, O.PHI_VARIANCE])
def test_phi_bar_golden_through_projection(mode):
    z, s, f = 4.0, 0.05, 60.0
    cam = cam_identity(f=f)
    for beta, rho, phi in golden_phi():
        parts = one_particle([0, 0, z], [math.log(s)] * 3, beta=beta)
        pre = O.preprocess(parts, cam, O.Settings(rho=rho, phi_mode=mode), "f64")
        m = phi if mode == O.PHI_SCALE else math.sqrt(phi)
        s32 = math.exp(float(np.float32(math.log(s))))     # parameters are fp32
        sigma2 = (f * m * s32 / z) ** 2 + 0.3
        A, B, Cc = pre["cov2d"][:, 0]
        # rho enters through the fp32 settings struct (rel. error 1.5e-9 -> ~1e-9 in phi)
        assert abs(A - sigma2) <= 1e-8 * sigma2 and abs(Cc - sigma2) <= 1e-8 * sigma2 and abs(B) < 1e-15
        assert pre["uv"][0, 0] == cam.cx and pre["uv"][1, 0] == cam.cy


def test_beta2_and_rho0_bit_identical_to_gaussian_path():
    """PAPER.md:294 and Fig. 4 caption: phi-bar(2) = 1 exactly and
    rho = 0 reduces GES to Gaussian splatting for any beta."""
    sc = gi.make_config(0)
    cam = sc.cameras[0]
    g = O.preprocess(sc.particles, cam, O.Settings(gaussian_only=1), "f32")
    p2 = sc.particles.subset(slice(None))
    p2.beta[:] = 2.0
    b2 = O.preprocess(p2, cam, O.Settings(), "f32")
    r0 = O.preprocess(sc.particles, cam, O.Settings(rho=0.0), "f32")
    for k in ("depth", "uv", "conic", "cov2d", "kappa", "rgb", "radius", "rect", "tiles", "status", "flags"):
        assert np.array_equal(g[k], b2[k]), k
        assert np.array_equal(g[k], r0[k]), k
    # and beta != 2 really changes the footprint (phi-bar > 1 for beta > 2)
    p8 = sc.particles.subset(slice(None))
    p8.beta[:] = 8.0
    b8 = O.preprocess(p8, cam, O.Settings(), "f32")
    vis = (g["status"] == 0) & (b8["status"] == 0)
    assert np.all(b8["cov2d"][0, vis] > g["cov2d"][0, vis])


# --------------------------------------------------------------------------
# Sigma = R S S^T R^T (S scaled by phi-bar) and EWA Sigma' = J W Sigma W^T J^T
# --------------------------------------------------------------------------
def _numeric_jacobian(tcam, fx, fy):
    def proj(t):
        return np.array([fx * t[0] / t[2], fy * t[1] / t[2]])
    J = np.zeros((2, 3))
    for k in range(3):
        h = 1e-6 * max(1.0, abs(tcam[k]))
        e = np.zeros(3)
        e[k] = h
        J[:, k] = (proj(tcam + e) - proj(tcam - e)) / (2 * h)
    return J


@pytest.mark.parametrize("mode", [O.PHI_SCALE, O.PHI_VARIANCE])
def test_covariance_and_ewa_against_independent_construction(mode):
    rng = np.random.default_rng(7)
    cam = gi.make_config(2).cameras[3]
    P = 64
    mean = rng.normal(0, 0.3, (3, P))
    log_scale = rng.normal(-3.0, 0.5, (3, P))
    quat = rng.standard_normal((4, P))
    beta = rng.uniform(0.5, 8.0, P)
    parts = gi.Particles(*(np.ascontiguousarray(a, np.float32) for a in
                           (mean, log_scale, quat, rng.normal(0, 1, P), rng.normal(0, 0.3, (3, P)), beta)), 0)
    rho = 0.1
    pre = O.preprocess(parts, cam, O.Settings(rho=rho, phi_mode=mode), "f64")
    W = cam.R.astype(np.float64)
    for i in range(P):
        if pre["status"][i] != 0:
            continue
        q = parts.quat[:, i].astype(np.float64)
        Rq = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()   # scipy: (x, y, z, w)
        phi = 2.0 / (1.0 + math.exp(-(rho * float(parts.beta[i]) - 2 * rho)))
        m = phi if mode == O.PHI_SCALE else math.sqrt(phi)
        S = np.diag(np.exp(parts.log_scale[:, i].astype(np.float64)) * m)
        Sigma = Rq @ S @ S.T @ Rq.T
        tcam = W @ parts.mean[:, i].astype(np.float64) + cam.t.astype(np.float64)
        lim = 1.3 * 0.5 * cam.width / cam.fx
        if abs(tcam[0] / tcam[2]) > lim or abs(tcam[1] / tcam[2]) > lim:
            continue
        J = _numeric_jacobian(tcam, cam.fx, cam.fy)
        cov = J @ W @ Sigma @ W.T @ J.T + 0.3 * np.eye(2)
        got = pre["cov2d"][:, i]
        scale = abs(cov).max()
        assert np.allclose(got, [cov[0, 0], cov[0, 1], cov[1, 1]], rtol=0, atol=1e-7 * scale), (i, got, cov)
        inv = np.linalg.inv(cov)
        assert np.allclose(pre["conic"][:, i], [inv[0, 0], inv[0, 1], inv[1, 1]], rtol=1e-7, atol=0)
        u = cam.fx * tcam[0] / tcam[2] + cam.cx
        v = cam.fy * tcam[1] / tcam[2] + cam.cy
        assert abs(pre["uv"][0, i] - u) < 1e-9 and abs(pre["uv"][1, i] - v) < 1e-9
        lam = np.linalg.eigvalsh(cov).max()
        mid = 0.5 * (cov[0, 0] + cov[1, 1])
        if mid * mid - np.linalg.det(cov) > 0.2:   # away from the 0.1 floor reading (R7)
            assert pre["radius"][i] == math.ceil(3 * math.sqrt(lam))


def test_projection_properties():
    """SPEC.md:432-450 projection properties: doubling depth halves the std,
    camera roll leaves an isotropic footprint invariant."""
    cam = cam_identity(W=256, H=256, f=200.0)
    st = O.Settings(rho=0.0)
    s = 0.05
    a = O.preprocess(one_particle([0, 0, 2.0], [math.log(s)] * 3), cam, st, "f64")
    b = O.preprocess(one_particle([0, 0, 4.0], [math.log(s)] * 3), cam, st, "f64")
    va, vb = a["cov2d"][0, 0] - 0.3, b["cov2d"][0, 0] - 0.3
    assert abs(math.sqrt(va) / math.sqrt(vb) - 2.0) < 1e-12
    # roll: rotate the camera about its optical axis
    th = 0.7
    Rz = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]], np.float32)
    cam_r = gi.Camera(256, 256, 200.0, 200.0, 128.0, 128.0, 0.2, Rz, np.zeros(3, np.float32))
    p = one_particle([0.1, -0.05, 3.0], [math.log(s)] * 3)
    e0 = np.linalg.eigvalsh(_cov(O.preprocess(p, cam, st, "f64")))
    e1 = np.linalg.eigvalsh(_cov(O.preprocess(p, cam_r, st, "f64")))
    assert np.allclose(e0, e1, rtol=1e-3)  # EWA is a local linearisation: equal to first order


def _cov(pre):
    A, B, C = pre["cov2d"][:, 0]
    return np.array([[A, B], [B, C]])


# --------------------------------------------------------------------------
# Kernel value at sample pixels (Eq. 2 at beta = 2 is the textbook Gaussian;
# other beta enter only through phi-bar, Eq. 4-6)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("beta", [0.5, 1.0, 2.0, 4.0, 8.0])
@pytest.mark.parametrize("precision,tol", [("f64", 1e-12), ("f32", 2e-6)])
def test_kernel_value_isotropic_on_axis(beta, precision, tol):
    f, z, s, logit = 60.0, 4.0, 0.12, 0.3
    cam = cam_identity(W=64, H=64, f=f)
    bg = (0.1, 0.2, 0.3)
    st = O.Settings(rho=0.1, background=bg)
    sh0 = np.array([0.2, -0.4, 0.7])
    sh = sh0.reshape(3, 1)
    parts = one_particle([0, 0, z], [math.log(s)] * 3, logit=logit, beta=beta, sh=sh)
    out = O.render(parts, cam, st, precision)
    r32 = lambda v: float(np.float32(v))          # the particle/settings structs are fp32
    rho = r32(0.1)
    phi = 2.0 / (1.0 + math.exp(-(rho * beta - 2 * rho)))
    sig2 = (f * phi * math.exp(r32(math.log(s))) / z) ** 2 + 0.3
    kappa = 1.0 / (1.0 + math.exp(-r32(logit)))
    Y00 = 0.5 / math.sqrt(math.pi)
    rgb = np.maximum(Y00 * sh0.astype(np.float32).astype(np.float64) + 0.5, 0.0)
    bgc = np.array([np.float32(c) for c in bg], np.float64)
    sig = math.sqrt(sig2)
    for (py, px) in [(32, 32), (32, 35), (29, 31), (33, 38), (36, 36)]:
        d2 = (px + 0.5 - 32.0) ** 2 + (py + 0.5 - 32.0) ** 2
        if math.sqrt(d2) > 2.5 * sig:
            continue
        alpha = min(0.99, kappa * math.exp(-0.5 * d2 / sig2))
        expect = alpha * rgb + (1 - alpha) * bgc if alpha >= 1 / 255 else bgc
        got = out["image"][:, py, px]
        assert np.allclose(got, expect, rtol=0, atol=tol), (py, px, got, expect)


# --------------------------------------------------------------------------
# Eq. 3 discrete compositing invariants
# --------------------------------------------------------------------------
def _white(parts):
    p = parts.subset(slice(None))
    p.sh[:] = 0.0
    p.sh[0:3] = math.sqrt(math.pi)  # Y00 * sh = 0.5 -> rgb = 1 (up to fp32 rounding of sh)
    return p


def test_transmittance_plus_weights_is_one():
    sc = gi.make_config(0)
    cam = sc.cameras[0]
    out = O.render(_white(sc.particles), cam, O.Settings(), "f32")
    # rgb = const (degree-0 SH, same coefficients), bg = 0  =>  image = rgb * sum_i w_i
    rgb0 = float(out["pre"]["rgb"][0, out["pre"]["status"] == 0][0])
    assert abs(rgb0 - 1.0) < 1e-6
    s = out["image"][0] / rgb0 + out["final_T"]
    assert np.abs(s - 1.0).max() < 1e-12
    assert np.all(out["final_T"] <= 1.0) and np.all(out["final_T"] >= 0.0)
    # early termination keeps T >= 1e-4 (R12)
    assert out["final_T"].min() >= np.float32(1e-4)


def test_empty_scene_and_single_splat_at_center():
    cam = cam_identity(W=32, H=32, f=30.0)
    bg = (0.25, 0.5, 0.75)
    bgc = np.array([np.float32(c) for c in bg], np.float64)
    far = one_particle([0, 0, 0.1], [-2, -2, -2])  # behind the near plane
    out = O.render(far, cam, O.Settings(background=bg), "f64")
    assert np.allclose(out["image"], bgc[:, None, None], atol=0)
    # splat centred exactly on a pixel centre: d = 0, G = 1, alpha = kappa
    z = 3.0
    x = (16.5 - 16.0) * z / 30.0
    p = one_particle([x, x, z], [-2.5] * 3, logit=0.4)
    out = O.render(p, cam, O.Settings(background=bg), "f64")
    kappa = 1 / (1 + math.exp(-0.4))
    rgb = 0.5 / math.sqrt(math.pi) * 0.5 + 0.5
    assert np.allclose(out["image"][:, 16, 16], kappa * rgb + (1 - kappa) * bgc, atol=1e-12)


def test_two_overlapping_splats_front_to_back_closed_form():
    """Eq. 3 composites front to back: C = sum_i c_i a_i T_i with
    T_i = prod_{j<i} (1 - a_j), i in increasing depth.  Two splats centred on the
    same pixel centre (d = 0, G = 1, alpha = kappa) at depths z1 < z2 give
    C = k1 c1 + (1 - k1) k2 c2 + (1 - k1)(1 - k2) bg.  Walking the list back to
    front (or ordering by decreasing depth) gives k2 c2 + (1 - k2) k1 c1 + ... and
    fails; so does compositing in index order (the far splat has the lower index)."""
    cam = cam_identity(W=32, H=32, f=30.0)
    bg = (0.1, 0.2, 0.3)
    bgc = np.array([np.float32(c) for c in bg], np.float64)
    z1, z2 = 3.0, 5.0
    x1, x2 = (16.5 - 16.0) * z1 / 30.0, (16.5 - 16.0) * z2 / 30.0
    sh_far = np.array([[0.9], [-0.6], [0.1]])
    sh_near = np.array([[-0.7], [0.8], [0.3]])
    mean = np.array([[x2, x1], [x2, x1], [z2, z1]])      # index 0 = far, index 1 = near
    f32 = lambda a: np.ascontiguousarray(np.asarray(a, np.float64), np.float32)
    parts = gi.Particles(f32(mean), f32(np.full((3, 2), -2.5)), f32(np.tile([[1.0], [0], [0], [0]], (1, 2))),
                         f32([-0.2, 0.4]), f32(np.hstack([sh_far, sh_near])), f32([2.0, 2.0]), 0)
    out = O.render(parts, cam, O.Settings(background=bg), "f64")
    r32 = lambda v: np.asarray(v, np.float32).astype(np.float64)
    k_far, k_near = 1 / (1 + math.exp(-r32(-0.2))), 1 / (1 + math.exp(-r32(0.4)))
    Y00 = 0.5 / math.sqrt(math.pi)
    c_far, c_near = Y00 * r32(sh_far[:, 0]) + 0.5, Y00 * r32(sh_near[:, 0]) + 0.5
    front_to_back = k_near * c_near + (1 - k_near) * k_far * c_far + (1 - k_near) * (1 - k_far) * bgc
    back_to_front = k_far * c_far + (1 - k_far) * k_near * c_near + (1 - k_near) * (1 - k_far) * bgc
    got = out["image"][:, 16, 16]
    assert np.abs(front_to_back - back_to_front).min() > 1e-2   # the two orders are distinguishable
    assert np.allclose(got, front_to_back, rtol=0, atol=1e-12), (got, front_to_back, back_to_front)
    assert abs(out["final_T"][16, 16] - (1 - k_near) * (1 - k_far)) < 1e-12
    assert out["n_contrib"][16, 16] == 2


def test_permutation_invariance_and_convexity():
    sc = gi.make_config(0, P=400)
    cam = sc.cameras[0]
    a = O.render(sc.particles, cam, O.Settings(), "f64")
    perm = np.random.default_rng(3).permutation(sc.particles.P)
    b = O.render(sc.particles.subset(perm), cam, O.Settings(), "f64")
    assert np.abs(a["image"] - b["image"]).max() < 1e-12
    assert a["image"].min() >= 0.0 and a["image"].max() <= 1.0


def test_log_spec_accuracy_and_powers_of_two():
    x = np.exp(np.linspace(1e-6, 12.0, 400001)).astype(np.float32)
    x = x[x > 1]
    y = O.log_spec(x).astype(np.float64)
    ref = np.log(x.astype(np.float64))
    ulp = np.spacing(ref.astype(np.float32)).astype(np.float64)
    assert (np.abs(y - ref) / ulp).max() <= 3.0
    k = np.arange(1, 20)
    p2 = O.log_spec((2.0 ** k).astype(np.float32)).astype(np.float64)
    assert np.allclose(p2, k * math.log(2.0), rtol=0, atol=1e-6)


def _alpha_image(pre, i, W, H):
    """kappa exp(-Q/2) of particle i at every pixel centre (x + 0.5, y + 0.5), fp64."""
    px, py = np.meshgrid(np.arange(W) + 0.5, np.arange(H) + 0.5)
    ca, cb, cc = pre["conic"][:, i].astype(np.float64)
    dx, dy = float(pre["uv"][0, i]) - px, float(pre["uv"][1, i]) - py
    q = ca * dx * dx + cc * dy * dy + 2.0 * cb * dx * dy
    return float(pre["kappa"][i]) * np.exp(-0.5 * q)


def test_rect_holds_every_pixel_that_reaches_the_alpha_threshold():
    """R10: a pixel outside rect_i's tiles never sees alpha_i >= 1/255, and the
    rect is no wider than the 0.98/255 box needs (brute force over all pixels)."""
    sc = gi.random_small_scene(11, P=80, W=192, H=128, log_scale_mu=-1.7, kappa_max=0.99)
    cam = sc.cameras[0]
    pre = O.preprocess(sc.particles, cam, O.Settings(), "f32")
    W, H = cam.width, cam.height
    n_vis = n_tight = 0
    for i in range(sc.particles.P):
        if pre["status"][i] not in (O.VISIBLE, O.OFFSCREEN):
            continue
        a = _alpha_image(pre, i, W, H)
        x0, y0, x1, y1 = pre["rect"][:, i]
        inside = np.zeros((H, W), bool)
        inside[16 * y0:16 * y1, 16 * x0:16 * x1] = True
        assert a[~inside].max(initial=0.0) < 1.0 / 255, i
        q = 2.0 * math.log(255.0 * float(pre["kappa"][i]) / 0.98) if pre["kappa"][i] > 0.98 / 255 else 0.0
        ex, ey = math.sqrt(q * float(pre["cov2d"][0, i])), math.sqrt(q * float(pre["cov2d"][2, i]))
        u, v = float(pre["uv"][0, i]), float(pre["uv"][1, i])
        unclipped = u - ex > 0 and u + ex < W and v - ey > 0 and v + ey < H
        if pre["status"][i] == O.VISIBLE:
            n_vis += 1
            if not unclipped:
                continue
            n_tight += 1
            # tight: no rect edge tile column/row lies beyond the pixels that
            # reach alpha >= 0.25/255 (the pixel grid is within half a pixel of
            # the ellipse's extreme points; sigma >= sqrt(0.3) px after dilation)
            ys, xs = np.nonzero(a >= 0.25 / 255)
            assert ys.size > 0
            assert x0 >= xs.min() // 16 and x1 - 1 <= xs.max() // 16, i
            assert y0 >= ys.min() // 16 and y1 - 1 <= ys.max() // 16, i
        else:
            assert a.max() < 1.0 / 255
    assert n_vis > 40 and n_tight > 20, (n_vis, n_tight)


def test_rect_membership_equals_all_particles_in_all_tiles():
    """Eq. 3 with the alpha skip sums over ALL particles; restricting each to its
    rect tiles (R10) or to tiles that reach the threshold (R8 'exact') changes
    nothing: bit-identical images, gradients equal to 1e-12."""
    sc = gi.random_small_scene(12, P=120, W=96, H=64, log_scale_mu=-1.3, kappa_max=0.99)
    cam = sc.cameras[0]
    g = gi.upstream_grad(sc.seed, 0, cam.width, cam.height)
    outs = {m: O.render_and_grad(sc.particles, cam, O.Settings(), g, membership=m)
            for m in ("rect", "all", "exact")}
    a = outs["rect"]
    assert a["list"].size < outs["all"]["list"].size
    for m in ("all", "exact"):
        b = outs[m]
        assert np.array_equal(a["image"], b["image"]), m
        # n_contrib is a position in the tile's list, so only its zero set is shared
        assert np.array_equal(a["n_contrib"] > 0, b["n_contrib"] > 0), m
        assert np.array_equal(a["final_T"], b["final_T"]), m
        for k in a["grads"]:
            assert np.allclose(a["grads"][k], b["grads"][k], rtol=1e-12, atol=1e-12), (m, k)


# --------------------------------------------------------------------------
# Keys, sort, lists: numpy brute force on tiny inputs
# --------------------------------------------------------------------------
def test_keys_and_lists_bruteforce():
    sc = gi.make_config(0, P=300)
    cam = sc.cameras[0]
    pre = O.preprocess(sc.particles, cam, O.Settings(), "f32")
    keys, vals = O.pairs_sorted(pre, membership="rect")
    tx = pre["tiles_x"]
    db = pre["depth"].view(np.uint32)
    ek, ev = [], []
    for i in range(sc.particles.P):
        if pre["status"][i] != 0:
            continue
        x0, y0, x1, y1 = pre["rect"][:, i]
        for y in range(y0, y1):
            for x in range(x0, x1):
                ek.append((int(y * tx + x) << 32) | int(db[i]))
                ev.append(i)
    ek, ev = np.array(ek, np.uint64), np.array(ev, np.int32)
    o = np.lexsort((ev, ek))
    assert np.array_equal(keys, ek[o]) and np.array_equal(vals, ev[o])
    offsets, lst = O.tile_lists(pre, membership="rect")
    tiles = (keys >> np.uint64(32)).astype(np.int64)
    for t in range(tx * pre["tiles_y"]):
        sel = vals[tiles == t]
        assert np.array_equal(lst[offsets[t]:offsets[t + 1]], sel)
    # ranges by linear scan == offsets
    ranges = np.searchsorted(tiles, np.arange(tx * pre["tiles_y"] + 1))
    assert np.array_equal(ranges, offsets)


# --------------------------------------------------------------------------
# Adjoints vs central finite differences (all-fp64 pipeline)
# --------------------------------------------------------------------------
def _fd_check(scene, st, n_checks=None, rel=1e-5, seed=0):
    cam = scene.cameras[0]
    parts = scene.particles
    O.set_amb_margin(1e-3)
    try:
        base = O.render(parts, cam, st, "f64")
    finally:
        O.set_amb_margin(0.0)
    g = gi.upstream_grad(seed, 0, cam.width, cam.height).astype(np.float64)
    g[:, base["amb"] != 0] = 0.0   # never straddle a skip/stop/clamp decision
    pre = base["pre"]
    g2d = O.render_bwd(pre, cam, st, base["offsets"], base["list"], g)
    grads = O.backward_particles(parts, cam, st, g2d, pre["status"], pre["flags"])
    fails = []
    names = ("mean", "log_scale", "quat", "opacity_logit", "sh", "beta")
    for n in names:
        arr = getattr(parts, n)
        ga = grads[n]
        for idx in np.ndindex(arr.shape):
            i = idx[-1]
            if pre["status"][i] != 0:
                continue
            p64 = gi.Particles(*(np.array(getattr(parts, m), np.float64) for m in names[:5]),
                               np.array(parts.beta, np.float64), parts.sh_degree)
            x0 = float(getattr(p64, n)[idx])
            h = 1e-6 * max(1.0, abs(x0))
            getattr(p64, n)[idx] = x0 + h
            lp = O.loss_f64(p64, cam, st, g)
            getattr(p64, n)[idx] = x0 - h
            lm = O.loss_f64(p64, cam, st, g)
            fd = (lp - lm) / (2 * h)
            an = float(ga[idx])
            if abs(fd - an) > rel * max(abs(fd), abs(an)) + 1e-8:
                fails.append((n, idx, an, fd))
    assert not fails, fails[:10]
    return grads


@pytest.mark.parametrize("seed,deg,mode", [(1, 0, O.PHI_SCALE), (2, 1, O.PHI_SCALE), (3, 3, O.PHI_VARIANCE),
                                           (4, 3, O.PHI_SCALE)])
def test_gradients_finite_differences(seed, deg, mode):
    sc = gi.random_small_scene(seed, P=5, W=32, H=32, sh_degree=deg, kappa_max=0.6)
    st = O.Settings(rho=0.1, phi_mode=mode, background=(0.1, 0.3, 0.2))
    _fd_check(sc, st)


def test_gradients_fd_large_rho_and_off_axis_camera():
    sc = gi.random_small_scene(11, P=4, W=48, H=32, sh_degree=2, kappa_max=0.6)
    cam = sc.cameras[0]
    R, t = gi.look_at((0.4, -0.3, -0.5), target=(0.0, 0.0, 4.0))
    sc.cameras[0] = gi.Camera(cam.width, cam.height, cam.fx, cam.fy * 1.1, cam.cx + 1.5, cam.cy - 2.0, 0.2, R, t)
    _fd_check(sc, O.Settings(rho=0.5))


def test_beta_gradient_identity_and_zero_cases():
    """dL/dbeta = rho phi'(beta)/phi ... : with s_eff = s*m(beta),
    dL/dbeta = (dm/dbeta / m) * sum_k dL/dlog s_k; m = phi (SCALE) gives
    rho (1 - phi/2), m = sqrt(phi) gives half that (Eq. 6 derivative)."""
    sc = gi.make_config(0, P=500)
    cam = sc.cameras[0]
    g = gi.upstream_grad(sc.seed, 0, cam.width, cam.height)
    for mode, fac in ((O.PHI_SCALE, 1.0), (O.PHI_VARIANCE, 0.5)):
        st = O.Settings(rho=0.1, phi_mode=mode)
        r = O.render_and_grad(sc.particles, cam, st, g)
        rho = float(np.float32(0.1))   # settings carry fp32 rho
        phi = 2.0 / (1.0 + np.exp(-(rho * sc.particles.beta.astype(np.float64) - 2 * rho)))
        expect = fac * rho * (1 - phi / 2) * r["grads"]["log_scale"].sum(axis=0)
        assert np.allclose(r["grads"]["beta"], expect, rtol=1e-10, atol=1e-14)
    r0 = O.render_and_grad(sc.particles, cam, O.Settings(rho=0.0), g)
    assert np.all(r0["grads"]["beta"] == 0.0)
    rz = O.render_and_grad(sc.particles, cam, O.Settings(), np.zeros_like(g))
    for v in rz["grads"].values():
        assert np.all(v == 0.0)


def test_sh_gradient_linear_in_upstream():
    sc = gi.make_config(0, P=300)
    cam = sc.cameras[0]
    g = gi.upstream_grad(sc.seed, 0, cam.width, cam.height).astype(np.float64)
    a = O.render_and_grad(sc.particles, cam, O.Settings(), g)["grads"]["sh"]
    b = O.render_and_grad(sc.particles, cam, O.Settings(), 2.5 * g)["grads"]["sh"]
    assert np.allclose(b, 2.5 * a, rtol=1e-12, atol=1e-15)


# --------------------------------------------------------------------------
# SH basis: orthonormal on the sphere (pins constants and polynomials)
# --------------------------------------------------------------------------
def test_sh_basis_orthonormal():
    n = 24
    xg, wg = np.polynomial.legendre.leggauss(n)        # cos(theta)
    phis = np.arange(2 * n) * (2 * math.pi / (2 * n))  # exact for trig degree < 2n
    Gram = np.zeros((16, 16))
    for ct, w in zip(xg, wg):
        st_ = math.sqrt(1 - ct * ct)
        for ph in phis:
            d = (st_ * math.cos(ph), st_ * math.sin(ph), ct)
            Y = O.sh_basis(d, 16)
            Gram += w * (2 * math.pi / (2 * n)) * np.outer(Y, Y)
    assert np.abs(Gram - np.eye(16)).max() < 1e-12
    # DC constant 1/(2 sqrt(pi)); fp32 KEYSPEC basis agrees with fp64 to fp32 precision
    assert abs(O.sh_basis((0, 0, 1), 1)[0] - 0.28209479177387814) < 1e-16
    d = np.array([0.3, -0.5, 0.8])
    d /= np.linalg.norm(d)
    assert np.allclose(O.sh_basis(d.astype(np.float32), 16, "f32"), O.sh_basis(d, 16), rtol=2e-6, atol=1e-7)


def test_ambiguity_flags_are_rare_on_config0():
    sc = gi.make_config(0)
    out = O.render(sc.particles, sc.cameras[0], O.Settings(), "f32")
    assert (out["amb"] != 0).mean() < 1e-3


def test_exact_membership_changes_nothing_but_the_lists():
    """R8: dropping (tile, particle) pairs that cannot reach alpha >= 0.98/255
    anywhere in the tile leaves images and gradients exactly unchanged, and
    the kept pairs keep their (tile, depth, index) order."""
    sc = gi.make_config(1, P=4000)
    cam = sc.cameras[0]
    g = gi.upstream_grad(sc.seed, 0, cam.width, cam.height)
    a = O.render_and_grad(sc.particles, cam, O.Settings(), g, membership="rect")
    b = O.render_and_grad(sc.particles, cam, O.Settings(), g, membership="exact")
    assert np.array_equal(a["image"], b["image"])
    assert np.array_equal(a["n_contrib"] > 0, b["n_contrib"] > 0)
    for k in a["grads"]:
        assert np.allclose(a["grads"][k], b["grads"][k], rtol=1e-12, atol=1e-12), k
    kr, vr = O.pairs_sorted(a["pre"], membership="rect")
    ke, ve = O.pairs_sorted(a["pre"], membership="exact")
    assert 0 < ke.size < kr.size
    pos = {(int(k), int(v)): n for n, (k, v) in enumerate(zip(kr, vr))}
    idx = np.array([pos[(int(k), int(v))] for k, v in zip(ke, ve)])
    assert np.all(np.diff(idx) > 0)   # a subsequence of the rect order
    # membership really is the alpha test: every dropped pair's particle is at most
    # 0.98/255 at the tile's nearest pixel centre (brute force over the tile's pixels)
    pre = a["pre"]
    dropped = set(zip(kr.tolist(), vr.tolist())) - set(zip(ke.tolist(), ve.tolist()))
    tx_n = pre["tiles_x"]
    for k, i in list(dropped)[:200]:
        t = k >> 32
        ty, tx = divmod(t, tx_n)
        px, py = np.meshgrid(np.arange(16) + 16 * tx + 0.5, np.arange(16) + 16 * ty + 0.5)
        ca, cb, cc = pre["conic"][:, i].astype(np.float64)
        dx, dy = pre["uv"][0, i] - px, pre["uv"][1, i] - py
        alpha = pre["kappa"][i] * np.exp(-0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy)
        assert alpha.max() < 0.99 / 255


# --------------------------------------------------------------------------
# R19 magnitudes: sum over terms of |term| (the condition-number denominators)
# --------------------------------------------------------------------------
def test_r19_magnitudes_bound_the_gradients():
    """|sum| <= sum |terms| for every S5a plane and every parameter gradient entry
    (triangle inequality); the magnitudes are homogeneous of degree 1 in dL/dimage
    and depend only on |dL/dimage| per term; with dL/dimage >= 0 and a black
    background the colour planes have no cancellation (each term alpha T g >= 0)
    and equal their sums exactly."""
    sc = gi.make_config(0, P=600)
    cam = sc.cameras[0]
    st = O.Settings()
    g = gi.upstream_grad(sc.seed, 0, cam.width, cam.height).astype(np.float64)
    base = O.render(sc.particles, cam, st, "f32")
    pre = base["pre"]
    g2d, gabs = O.render_bwd(pre, cam, st, base["offsets"], base["list"], g, with_abs=True)
    assert np.array_equal(g2d, O.render_bwd(pre, cam, st, base["offsets"], base["list"], g))
    assert np.all(np.abs(g2d) <= gabs[:10] * (1 + 1e-12) + 1e-300)
    assert np.all(gabs[10:] >= 0) and np.all(gabs[10:] <= 1e-3 * gabs[:10] + 1e-300)
    scale = O.grad_error_scale(sc.particles, cam, st, g2d, gabs, pre["status"], pre["flags"])
    grads = O.backward_particles(sc.particles, cam, st, g2d, pre["status"], pre["flags"])
    for n in grads:
        assert np.all(np.abs(grads[n]) <= scale["round"][n] * (1 + 1e-12) + 1e-300), n
    g2d2, gabs2 = O.render_bwd(pre, cam, st, base["offsets"], base["list"], 2.0 * g, with_abs=True)
    assert np.allclose(gabs2, 2.0 * gabs, rtol=1e-13, atol=0)
    gp = np.abs(g)
    g2dp, gabsp = O.render_bwd(pre, cam, st, base["offsets"], base["list"], gp, with_abs=True)
    assert np.array_equal(g2dp[6:9], gabsp[6:9])
    # the colour planes' sensitivity is exact: each term alpha T g moves by (eps_alpha + eps_T)
    assert np.all(gabsp[16:19] >= 2e-6 * gabsp[6:9])
    # S5b over magnitudes: one plane, one single-term chain (opacity: dk kappa (1 - kappa))
    e = np.zeros_like(g2d)
    e[5] = gabs[5]
    m = O.grad_magnitude(sc.particles, cam, st, e, pre["status"], pre["flags"])
    ref = O.backward_particles(sc.particles, cam, st, e, pre["status"], pre["flags"])
    assert np.allclose(m["opacity_logit"], np.abs(ref["opacity_logit"]), rtol=1e-15, atol=0)
    assert np.all(m["sh"] == 0) and np.all(m["mean"] == 0)


def test_r19_single_isotropic_splat_has_no_cancellation():
    """One isotropic splat (b = 0), one pixel with a nonnegative upstream gradient,
    black background: every S5a plane is a single term, so sum|terms| = |sum|."""
    cam = cam_identity(W=32, H=32, f=30.0)
    z = 3.0
    p = one_particle([0.0, 0.0, z], [-2.2] * 3, logit=0.3)   # on the axis: conic b = 0 exactly
    st = O.Settings()
    base = O.render(p, cam, st, "f32")
    g = np.zeros((3, 32, 32))
    g[:, 16, 15] = [0.4, 1.1, 0.7]
    g2d, gabs = O.render_bwd(base["pre"], cam, st, base["offsets"], base["list"], g, with_abs=True)
    assert np.abs(g2d[:9]).min() > 0
    assert np.allclose(np.abs(g2d[:9]), gabs[:9], rtol=1e-14, atol=0)
    # one splat, T = 1 exactly: the colour terms move only with alpha (eps_alpha = 2e-6 + 6e-7 |q|)
    assert np.all(gabs[16:19] > 2e-6 * gabs[6:9]) and np.all(gabs[16:19] < 1e-4 * gabs[6:9])


def test_definitional_lists_on_sampled_tiles_match_the_c_enumeration():
    """bench.py's definitional sample builds the 'all' membership of a few tiles
    directly (every particle, (depth, index) order); it equals the C brute force."""
    sc = gi.make_config(0, P=300)
    cam = sc.cameras[0]
    pre = O.preprocess(sc.particles, cam, O.Settings(), "f32")
    T = pre["tiles_x"] * pre["tiles_y"]
    mask = np.zeros(T, np.uint8)
    mask[[3, 50, 200]] = 1
    off, lst = O.tile_lists(pre, mask, membership="all")
    full_off, full_lst = O.tile_lists(pre, np.ones(T, np.uint8), membership="all")
    for t in range(T):
        got = lst[off[t]:off[t + 1]]
        want = full_lst[full_off[t]:full_off[t + 1]] if mask[t] else full_lst[:0]
        assert np.array_equal(got, want), t


def test_r18_both_branches_skip_decision_closed_form():
    """R18: a splat centred on a pixel centre (d = 0, G = 1, alpha = kappa)
    with kappa = 1/255 to fp32 rounding puts the pixel's skip decision inside the fp32
    error bound: the oracle flags the pixel, and its both-branch alternative is the
    other outcome in closed form -- one of (image, alternative) is the background
    (skipped) and the other kappa c + (1 - kappa) bg (composited); a pixel with no
    ambiguous decision has no alternative (NaN)."""
    cam = cam_identity(W=32, H=32, f=30.0)
    bg = (0.1, 0.2, 0.3)
    bgc = np.array([np.float32(c) for c in bg], np.float64)
    z = 4.0
    x = (16.5 - 16.0) * z / 30.0
    kappa = 1.0 / 255.0
    sh = np.array([[0.9], [-0.6], [0.1]])
    f32 = lambda a: np.ascontiguousarray(np.asarray(a, np.float64), np.float32)
    parts = gi.Particles(f32([[x], [x], [z]]), f32(np.full((3, 1), -2.5)), f32([[1.0], [0], [0], [0]]),
                         f32([math.log(kappa / (1 - kappa))]), f32(sh), f32([2.0]), 0)
    st = O.Settings(background=bg)
    pre = O.preprocess(parts, cam, st, "f32")
    offsets, lst = O.tile_lists(pre)
    ref = O.render_fwd(pre, cam, st, offsets, lst)
    assert ref["amb"][16, 16] != 0
    alt = O.render_fwd_alternatives(pre, cam, st, offsets, lst, ref["amb"], n_alt=2)
    k = float(pre["kappa"][0])
    assert abs(k - kappa) < 1e-6 * kappa
    c = pre["rgb"][:, 0].astype(np.float64)
    composited, skipped = k * c + (1 - k) * bgc, bgc
    pair = [ref["image"][:, 16, 16], alt[0][:, 16, 16]]
    assert any(np.allclose(pair[i], composited, rtol=0, atol=1e-12) and np.allclose(pair[1 - i], skipped, rtol=0,
                                                                                       atol=1e-12) for i in (0, 1))
    assert np.isnan(alt[1][:, 16, 16]).all()          # one ambiguous decision only
    assert np.isnan(alt[0][:, 0, 0]).all() and ref["amb"][0, 0] == 0   # unflagged pixel


def test_sh_gradient_factorises_per_view():
    """The SH part of S5b is the outer product Y_k(u) * dL/drgb (zero through a clamped
    channel, R13) per view -- the identity the SH-factorised view-DP exchange rests on
    (DESIGN.md §8): the oracle's SH gradient against the pinned SH basis (orthonormal, above)
    evaluated at u = (mean - camera centre) / |.|, times its own S5a colour sums, for each of
    two views."""
    sc = gi.make_config(2, P=300, n_views=2)
    parts = sc.particles
    st = O.Settings(rho=sc.rho)
    K = parts.K
    total = np.zeros((3 * K, parts.P))
    for v, cam in enumerate(sc.cameras):
        pre = O.preprocess(parts, cam, st, "f32")
        offsets, lst = O.tile_lists(pre)
        g = gi.upstream_grad(sc.seed, v, cam.width, cam.height).astype(np.float64)
        g2d = O.render_bwd(pre, cam, st, offsets, lst, g)
        sh = O.backward_particles(parts, cam, st, g2d, pre["status"], pre["flags"])["sh"]
        total += sh
        R = np.asarray(cam.R, np.float64).reshape(3, 3)
        centre = -R.T @ np.asarray(cam.t, np.float64).reshape(3)
        vis = np.nonzero(pre["status"] == 0)[0]
        assert vis.size > 20
        want = np.zeros_like(sh)
        for i in vis:
            d = parts.mean[:, i].astype(np.float64) - centre
            Y = O.sh_basis(d / np.linalg.norm(d), K)
            for ch in range(3):
                if not (pre["flags"][i] >> ch) & 1:
                    want[ch::3, i] = Y * g2d[6 + ch, i]
        scale = np.abs(want).max()
        assert np.abs(sh - want).max() <= 1e-9 * scale
        assert np.all(sh[:, pre["status"] != 0] == 0.0)
    assert np.count_nonzero(total) > 0
