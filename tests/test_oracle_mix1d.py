"""Pins of the 1-D mixture / Theorem-1 oracle (oracle/mix1d.py; SURVEY.md §8(f)
NEXT-4), each against something other than the oracle's own formulas:
  * every model's gradient (mu, s, omega, beta; real and positive weights) against
    central finite differences of its MSE
  * GEF at beta = 2 is the Gaussian mixture ("reduces to");
    a DoG component is two Gaussian components (s and s / sqrt(nu)) subtracted;
    a LoG component equals its weight at the mean and vanishes at |x - mu| = s
  * the signals' integrals against their closed forms (sigma, sigma^2/4, sigma^3/6,
    2 sigma/pi, 2 (1 - e^{-sigma/2}), sigma sqrt(2 pi)) by fine Riemann sums
  * Adam's first step is -lr g / (|g| + eps) (bias correction)
  * Theorem 1: the incomplete-gamma closed form against scipy.integrate.quad of the
    proof's integrals; beta = 2 equals the proof's Gaussian error (erf form); for
    every alpha on a grid some beta gives a strictly smaller error (the theorem)
"""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import mix1d as M


def _theta(rng, N, model):
    mu = rng.uniform(-1.5, 1.5, N)
    s = rng.uniform(0.2, 0.6, N)
    om = rng.normal(0.0, 0.5, N)
    beta = 1.7 if model == "gef" else 2.0
    return np.concatenate([mu, s, om, [beta]])


@pytest.mark.parametrize("model", M.MODELS)
@pytest.mark.parametrize("positive", [False, True])
def test_gradients_finite_differences(model, positive):
    rng = np.random.default_rng(3 + M.MODELS.index(model))
    N = 4
    x = M.grid(-2.0, 2.0, 301) + 1e-3       # no sample exactly on a mean
    y = M.signal("square", x, 1.0)
    th = _theta(rng, N, model)
    _, g = M.loss_and_grad(model, positive, th, N, x, y)
    h = 1e-6
    for k in range(3 * N + 1):
        if model != "gef" and k == 3 * N:
            assert g[k] == 0.0
            continue
        tp, tm = th.copy(), th.copy()
        tp[k] += h
        tm[k] -= h
        fd = (M.loss_and_grad(model, positive, tp, N, x, y)[0] - M.loss_and_grad(model, positive, tm, N, x, y)[0]) / (2 * h)
        assert abs(fd - g[k]) <= 1e-6 * max(1.0, abs(fd)), (model, k, fd, g[k])


def test_gef_beta2_is_the_gaussian_mixture():
    rng = np.random.default_rng(5)
    N = 6
    x = M.grid(-2.0, 2.0, 257)
    th = _theta(rng, N, "gmm")
    th[3 * N] = 2.0
    assert np.allclose(M.predict("gef", True, th, N, x), M.predict("gmm", True, th, N, x), rtol=1e-12, atol=1e-14)


def test_dog_is_two_gaussians_and_log_zeros():
    rng = np.random.default_rng(6)
    N = 3
    x = M.grid(-2.0, 2.0, 129)
    th = _theta(rng, N, "dog")
    narrow = th.copy()
    narrow[N:2 * N] = th[N:2 * N] / math.sqrt(M.NU)
    dog = M.predict("dog", False, th, N, x)
    assert np.allclose(dog, M.predict("gmm", False, th, N, x) - M.predict("gmm", False, narrow, N, x), atol=1e-14)
    one = np.array([0.3, 0.5, 0.7, 2.0])    # mu, s, omega, beta (N = 1, real weights)
    at = np.array([0.3, 0.3 + 0.5, 0.3 - 0.5])
    v = M.predict("log", False, one, 1, at)
    assert abs(v[0] - 0.7) < 1e-14 and abs(v[1]) < 1e-14 and abs(v[2]) < 1e-14


@pytest.mark.parametrize("kind,integral", [
    ("square", lambda s: s), ("triangle", lambda s: s * s / 4), ("parabolic", lambda s: s ** 3 / 6),
    ("half_sinusoid", lambda s: 2 * s / math.pi), ("exponential", lambda s: 2 * (1 - math.exp(-s / 2))),
    ("gaussian", lambda s: s * math.sqrt(2 * math.pi))])
def test_signal_integrals(kind, integral):
    width = 1.3
    x = M.grid(-12.0, 12.0, 2_400_001)
    y = M.signal(kind, x, width)
    got = y.sum() * (x[1] - x[0])
    assert abs(got - integral(width)) < 2e-5 * max(1.0, integral(width)), (got, integral(width))


def test_adam_first_step_is_sign():
    g = np.array([0.3, -2.0, 1e-5, -7.0])
    th, m, v = M.adam_step(np.zeros(4), g, np.zeros(4), np.zeros(4), 1, lr=0.01)
    # m-hat = g, v-hat = g^2: the step is -lr g / (|g| + eps), -lr sign(g) up to eps
    assert np.allclose(th, -0.01 * g / (np.abs(g) + 1e-8), rtol=1e-12)
    assert np.allclose(th[[0, 1, 3]], -0.01 * np.sign(g[[0, 1, 3]]), rtol=1e-6)


def test_fit_decreases_loss():
    rng = np.random.default_rng(9)
    N = 5
    x = M.grid(-2.0, 2.0, 256)
    y = M.signal("square", x, 1.0)
    th0 = _theta(rng, N, "gef")
    th0[2 * N:3 * N] = -1.0
    L0 = M.loss_and_grad("gef", True, th0, N, x, y)[0]
    th, _, _, L = M.fit("gef", True, th0, N, x, y, steps=200, lr=1e-2)
    assert L < 0.5 * L0


@pytest.mark.parametrize("alpha,beta", [(0.2, 0.7), (0.4, 2.0), (0.5, 3.5), (1.0, 8.0), (2.0, 1.2)])
def test_theorem1_closed_form_against_quadrature(alpha, beta):
    A, L = 1.3, 1.0
    f = lambda t: A * math.exp(-((t / alpha) ** beta))
    mid = integrate.quad(lambda t: A - f(t), 0.0, L / 2, epsabs=1e-13, epsrel=1e-12, limit=200)[0]
    tail = integrate.quad(f, L / 2, np.inf, epsabs=1e-13, epsrel=1e-12, limit=200)[0]
    assert abs(M.theorem1_errors(alpha, beta, A, L) - (2 * mid + 2 * tail)) < 1e-9


def test_theorem1_gaussian_and_the_claim():
    alphas = np.geomspace(0.05, 5.0, 40)
    EG = M.theorem1_gaussian_error(alphas)
    assert np.allclose(M.theorem1_errors(alphas, 2.0), EG, rtol=1e-12)
    betas = np.linspace(0.25, 16.0, 400)
    E = M.theorem1_errors(alphas[:, None], betas[None, :])
    assert np.all(E.min(axis=1) < EG)
    # and the minimising beta is not 2 (the Gaussian is never the best GEF here)
    best = betas[E.argmin(axis=1)]
    assert np.all(np.abs(best - 2.0) > 0.1)
