"""Pins of the oracle's exact GEF kernel (`Settings.kernel = 1`).

The paper's Eq. 2 defines the generalized exponential
G(x) = exp(-1/2 ((x - mu)^T Sigma^-1 (x - mu))^(beta/2)); the rasterizer of
§4.1 replaces it by a Gaussian of the phi-bar-scaled covariance (PAPER.md:284-288,
DESIGN.md R6).  The exact mode evaluates Eq. 2 per pixel on the projected,
dilated Sigma2D (no phi-bar).  Checked here against what the mathematics fixes:
  * closed form of one isotropic particle on the optical axis, beta in
    {0.5, 1, 2, 4, 8}: alpha = kappa exp(-1/2 (d^2 / sigma^2)^(beta/2))
  * beta = 2: Eq. 2 IS the Gaussian -- images and every non-beta gradient
    equal the Gaussian kernel's (rho = 0, phi-bar = 1)
  * the exact-mode rect holds every pixel that reaches alpha >= 1/255
    (brute force over all pixels), for beta in [0.5, 8]
  * every parameter gradient group, beta's direct term
    dG/dbeta = -1/4 G Q^(beta/2) ln Q included, against central finite
    differences of the all-fp64 pipeline
  * the KEYSPEC log on (0, 1) (the rect bound takes log(2 ln(255 kappa/0.98)))
"""
import math

import numpy as np
import pytest

import ges_inputs as gi
from oracle import oracle as O
from test_oracle_pins import _fd_check, cam_identity, one_particle

EXACT = O.KERNEL_EXACT_BETA


@pytest.mark.parametrize("beta", [0.5, 1.0, 2.0, 4.0, 8.0])
@pytest.mark.parametrize("precision,tol", [("f64", 1e-12), ("f32", 2e-6)])
def test_exact_kernel_value_isotropic_on_axis(beta, precision, tol):
    f, z, s, logit = 60.0, 4.0, 0.12, 0.3
    cam = cam_identity(W=64, H=64, f=f)
    bg = (0.1, 0.2, 0.3)
    st = O.Settings(rho=0.1, background=bg, kernel=EXACT)
    sh0 = np.array([0.2, -0.4, 0.7])
    parts = one_particle([0, 0, z], [math.log(s)] * 3, logit=logit, beta=beta, sh=sh0.reshape(3, 1))
    out = O.render(parts, cam, st, precision, membership="all")
    r32 = lambda v: float(np.float32(v))
    sig2 = (f * math.exp(r32(math.log(s))) / z) ** 2 + 0.3          # no phi-bar in Eq. 2
    kappa = 1.0 / (1.0 + math.exp(-r32(logit)))
    rgb = np.maximum(0.5 / math.sqrt(math.pi) * sh0.astype(np.float32).astype(np.float64) + 0.5, 0.0)
    bgc = np.array([np.float32(c) for c in bg], np.float64)
    hb = r32(beta) / 2.0
    n = 0
    for (py, px) in [(32, 32), (32, 35), (29, 31), (33, 38), (36, 36), (32, 41), (25, 30)]:
        q = ((px + 0.5 - 32.0) ** 2 + (py + 0.5 - 32.0) ** 2) / sig2
        alpha = min(0.99, kappa * math.exp(-0.5 * q ** hb))
        if abs(alpha - 1 / 255) < 1e-4:
            continue
        expect = alpha * rgb + (1 - alpha) * bgc if alpha >= 1 / 255 else bgc
        got = out["image"][:, py, px]
        assert np.allclose(got, expect, rtol=0, atol=tol), (py, px, got, expect)
        n += 1
    assert n >= 5


def test_exact_beta2_is_the_gaussian_kernel():
    sc = gi.random_small_scene(5, P=40, W=64, H=48, sh_degree=1, beta_range=(2.0, 2.0))
    cam = sc.cameras[0]
    g = gi.upstream_grad(5, 0, cam.width, cam.height)
    ex = O.render_and_grad(sc.particles, cam, O.Settings(rho=0.0, kernel=EXACT), g, membership="all")
    ga = O.render_and_grad(sc.particles, cam, O.Settings(rho=0.0), g, membership="all")
    assert np.allclose(ex["image"], ga["image"], rtol=0, atol=1e-12)
    for n in ("mean", "log_scale", "quat", "opacity_logit", "sh"):
        assert np.allclose(ex["grads"][n], ga["grads"][n], rtol=1e-10, atol=1e-13), n
    assert np.all(ga["grads"]["beta"] == 0.0)          # rho = 0: no phi-bar path
    assert np.any(ex["grads"]["beta"] != 0.0)          # Eq. 2's own beta dependence


def test_exact_rect_holds_every_pixel_that_reaches_the_alpha_threshold():
    sc = gi.random_small_scene(13, P=80, W=192, H=128, log_scale_mu=-2.2, kappa_max=0.99, beta_range=(0.5, 8.0))
    cam = sc.cameras[0]
    st = O.Settings(kernel=EXACT)
    pre = O.preprocess(sc.particles, cam, st, "f32")
    W, H = cam.width, cam.height
    px, py = np.meshgrid(np.arange(W) + 0.5, np.arange(H) + 0.5)
    n_vis = 0
    for i in range(sc.particles.P):
        if pre["status"][i] not in (O.VISIBLE, O.OFFSCREEN):
            continue
        ca, cb, cc = pre["conic"][:, i].astype(np.float64)
        dx, dy = float(pre["uv"][0, i]) - px, float(pre["uv"][1, i]) - py
        q = np.maximum(ca * dx * dx + cc * dy * dy + 2.0 * cb * dx * dy, 0.0)
        a = float(pre["kappa"][i]) * np.exp(-0.5 * q ** (float(sc.particles.beta[i]) / 2.0))
        x0, y0, x1, y1 = pre["rect"][:, i]
        inside = np.zeros((H, W), bool)
        inside[16 * y0:16 * y1, 16 * x0:16 * x1] = True
        assert a[~inside].max(initial=0.0) < 1.0 / 255, i
        n_vis += pre["status"][i] == O.VISIBLE
    assert n_vis > 30


@pytest.mark.parametrize("seed,deg", [(21, 0), (22, 1), (23, 3)])
def test_exact_gradients_finite_differences(seed, deg):
    sc = gi.random_small_scene(seed, P=5, W=32, H=32, sh_degree=deg, kappa_max=0.6, beta_range=(0.7, 6.0))
    st = O.Settings(rho=0.1, background=(0.1, 0.3, 0.2), kernel=EXACT)
    grads = _fd_check(sc, st)
    assert np.any(grads["beta"] != 0.0)


def test_exact_beta_gradient_has_no_phi_bar_term():
    """In the exact kernel beta enters only through Eq. 2's exponent: rho (which
    only scales phi-bar) changes neither the image nor any gradient."""
    sc = gi.random_small_scene(7, P=30, W=48, H=48, sh_degree=1)
    cam = sc.cameras[0]
    g = gi.upstream_grad(7, 0, cam.width, cam.height)
    a = O.render_and_grad(sc.particles, cam, O.Settings(rho=0.1, kernel=EXACT), g)
    b = O.render_and_grad(sc.particles, cam, O.Settings(rho=0.7, kernel=EXACT), g)
    assert np.array_equal(a["image"], b["image"])
    for n in a["grads"]:
        assert np.array_equal(a["grads"][n], b["grads"][n]), n


def test_log_spec_below_one():
    x = np.exp(np.linspace(-12.0, -1e-6, 200001)).astype(np.float32)
    x = x[(x < 1) & (x > 0)]
    y = O.log_spec(x).astype(np.float64)
    ref = np.log(x.astype(np.float64))
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    assert (np.abs(y - ref) / ulp).max() <= 3.0
