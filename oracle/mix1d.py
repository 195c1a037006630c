"""Plain fp64 numpy oracle of the 1-D mixture simulation and the Theorem-1
numerics.  TEST INFRASTRUCTURE ONLY (like oracle.py):
imported by tests/ and bench.py's baseline legs, never by the product package.

What it computes (PAPER.md Appendix "Numerical Simulation of Gradient-Based 1D
Mixtures", :606-745, and Theorem 1 with its proof, :555-603), with the readings
DESIGN.md R34-R37 lists where the paper is silent:
  signal           the six ground-truth signals of width sigma (:662-745): square,
                   triangle, parabolic, half sinusoid, exponential (all zero outside
                   (-sigma/2, sigma/2)) and Gaussian exp(-x^2 / (2 sigma^2))
  grid             x = linspace(x_lo, x_hi, n) (:628 "a linearly spaced tensor")
  mixture          Eq. (:633-658): GMM  sum w exp(-d^2 / (2 s^2 + eps)),
                   DoG  sum w (exp(-d^2 / (2 s^2 + eps)) - exp(-d^2 / (2 s^2 / nu + eps))), nu = 4,
                   LoG  sum w (1 - d^2 / s^2) exp(-d^2 / (2 s^2 + eps)),
                   GEF  sum w exp(-|d|^beta / (2 s^2 + eps)), one learnable beta (R34),
                   d = x - mu, eps = 1e-8; weights w = omega (real) or exp(omega)
                   (positive, R35)
  loss_and_grad    MSE = mean (h(x) - y)^2 and its hand-derived gradient in every
                   parameter (mu, s, omega per component, beta)
  adam_step        PyTorch's Adam (bias-corrected, eps outside the sqrt) (:628)
  fit              `steps` Adam steps from the given start; the loss at the end
  theorem1_errors  E_G(alpha) and E_GEF(alpha, beta) of the square wave (amplitude A,
                   width L) in closed form: with c = (L / (2 alpha))^beta,
                   int_0^{L/2} e^{-(t/alpha)^beta} dt = alpha/beta Gamma(1/beta) P(1/beta, c),
                   E = 2A (L/2 - that) + 2A alpha/beta Gamma(1/beta) Q(1/beta, c)  (:570-575)
Parameter layout of one run: [mu_0..mu_{N-1}, s_0.., omega_0.., beta].
"""
from __future__ import annotations

import math

import numpy as np
from scipy import special

EPS = 1e-8
NU = 4.0          # PAPER.md:651 "the variance ratio nu is fixed to be 4"
MODELS = ("gmm", "dog", "log", "gef")
SIGNALS = ("square", "triangle", "parabolic", "half_sinusoid", "exponential", "gaussian")


def grid(x_lo: float, x_hi: float, n: int) -> np.ndarray:
    """x_j = x_lo + j h, h = (x_hi - x_lo) / (n - 1)."""
    h = (x_hi - x_lo) / (n - 1)
    return x_lo + np.arange(n, dtype=np.float64) * h


def signal(kind: str, x: np.ndarray, width: float) -> np.ndarray:
    """The ground-truth signals of PAPER.md:662-745 (value 0 outside the open interval)."""
    x = np.asarray(x, np.float64)
    half = width / 2.0
    inside = (x > -half) & (x < half)
    if kind == "square":
        v = np.ones_like(x)
    elif kind == "triangle":
        v = half - np.abs(x)
    elif kind == "parabolic":
        v = half * half - x * x
    elif kind == "half_sinusoid":
        v = np.sin((x + half) * math.pi / width)
    elif kind == "exponential":
        v = np.exp(-np.abs(x))
    elif kind == "gaussian":
        return np.exp(-x * x / (2.0 * width * width))
    else:
        raise ValueError(kind)
    return np.where(inside, v, 0.0)


def split(theta: np.ndarray, N: int):
    theta = np.asarray(theta, np.float64)
    return theta[0:N], theta[N:2 * N], theta[2 * N:3 * N], float(theta[3 * N])


def weights(omega: np.ndarray, positive: bool):
    """(w, dw/domega)."""
    if positive:
        w = np.exp(omega)
        return w, w
    return omega, np.ones_like(omega)


def components(model: str, x: np.ndarray, mu, s, beta):
    """phi_i(x_j) and its partials d/dmu, d/ds (and d/dbeta for GEF), arrays [N][n]."""
    d = x[None, :] - mu[:, None]
    d2 = d * d
    D = 2.0 * s[:, None] ** 2 + EPS
    dD = 4.0 * s[:, None]                      # dD/ds
    zero = np.zeros_like(d)
    if model == "gmm":
        e = np.exp(-d2 / D)
        return e, e * 2.0 * d / D, e * d2 * dD / D ** 2, zero
    if model == "dog":
        D2 = 2.0 * s[:, None] ** 2 / NU + EPS
        e1, e2 = np.exp(-d2 / D), np.exp(-d2 / D2)
        return (e1 - e2, e1 * 2.0 * d / D - e2 * 2.0 * d / D2,
                e1 * d2 * dD / D ** 2 - e2 * d2 * (dD / NU) / D2 ** 2, zero)
    if model == "log":
        g2 = s[:, None] ** 2
        a = 1.0 - d2 / g2
        e = np.exp(-d2 / D)
        phi = a * e
        dmu = (2.0 * d / g2) * e + a * e * 2.0 * d / D
        ds = (2.0 * d2 / (g2 * s[:, None])) * e + a * e * d2 * dD / D ** 2
        return phi, dmu, ds, zero
    if model == "gef":
        ad = np.abs(d)
        nz = ad > 0.0
        lad = np.log(np.where(nz, ad, 1.0))
        p = np.where(nz, np.exp(beta * lad), 0.0)          # |d|^beta (beta > 0)
        e = np.exp(-p / D)
        # d|d|^beta/dmu = -beta |d|^(beta - 1) sign(d); d|d|^beta/dbeta = |d|^beta ln|d|; 0 at d = 0
        dmu = np.where(nz, e * beta * p / np.where(nz, ad, 1.0) * np.sign(d) / D, 0.0)
        ds = e * p * dD / D ** 2
        db = np.where(nz, -e * p * lad / D, 0.0)
        return e, dmu, ds, db
    raise ValueError(model)


def predict(model: str, positive: bool, theta, N: int, x):
    mu, s, om, beta = split(theta, N)
    w, _ = weights(om, positive)
    phi = components(model, np.asarray(x, np.float64), mu, s, beta)[0]
    return (w[:, None] * phi).sum(axis=0)


def loss_and_grad(model: str, positive: bool, theta, N: int, x, y):
    """MSE and its gradient in the run's parameter layout."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    mu, s, om, beta = split(theta, N)
    w, dw = weights(om, positive)
    phi, dmu, ds, db = components(model, x, mu, s, beta)
    r = (w[:, None] * phi).sum(axis=0) - y
    n = x.size
    L = float((r * r).sum() / n)
    c = 2.0 * r / n
    g = np.zeros(3 * N + 1)
    g[0:N] = (w[:, None] * dmu * c[None, :]).sum(axis=1)
    g[N:2 * N] = (w[:, None] * ds * c[None, :]).sum(axis=1)
    g[2 * N:3 * N] = (dw[:, None] * phi * c[None, :]).sum(axis=1)
    g[3 * N] = float((w[:, None] * db * c[None, :]).sum()) if model == "gef" else 0.0
    return L, g


def adam_step(theta, g, m, v, t: int, lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
    """torch.optim.Adam (t >= 1): theta - lr mhat / (sqrt(vhat) + eps)."""
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    return theta - lr * mh / (np.sqrt(vh) + eps), m, v


def fit(model: str, positive: bool, theta0, N: int, x, y, steps: int, lr: float = 1e-2,
        b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
    """`steps` Adam steps from theta0 (the beta slot is frozen for the non-GEF
    models: its gradient is 0).  Returns (theta, m, v, final loss)."""
    theta = np.array(theta0, np.float64)
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    for t in range(1, steps + 1):
        _, g = loss_and_grad(model, positive, theta, N, x, y)
        theta, m, v = adam_step(theta, g, m, v, t, lr, b1, b2, eps)
    return theta, m, v, loss_and_grad(model, positive, theta, N, x, y)[0]


def theorem1_errors(alpha, beta, A: float = 1.0, L: float = 1.0):
    """E_GEF(alpha, beta) of Theorem 1 in closed form via the
    regularised incomplete gamma functions; beta = 2 is E_G.  Broadcasts."""
    alpha = np.asarray(alpha, np.float64)
    beta = np.asarray(beta, np.float64)
    c = (L / (2.0 * alpha)) ** beta
    a = 1.0 / beta
    scale = alpha / beta * special.gamma(a)
    inner = scale * special.gammainc(a, c)       # int_0^{L/2} e^{-(t/alpha)^beta} dt
    tail = scale * special.gammaincc(a, c)       # int_{L/2}^inf
    return 2.0 * A * (L / 2.0 - inner) + 2.0 * A * tail


def theorem1_gaussian_error(alpha, A: float = 1.0, L: float = 1.0):
    """E_G of the proof with the error function: 2A (L/2 - a sqrt(pi)/2 erf(z)) + 2A a sqrt(pi)/2 erfc(z),
    z = L / (2 alpha)."""
    alpha = np.asarray(alpha, np.float64)
    z = L / (2.0 * alpha)
    k = alpha * math.sqrt(math.pi) / 2.0
    return 2.0 * A * (L / 2.0 - k * special.erf(z)) + 2.0 * A * k * special.erfc(z)
