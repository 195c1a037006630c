"""Plain fp64 numpy oracle of the image-loss front end.

TEST INFRASTRUCTURE ONLY (like oracle.py): imported by tests/ and bench.py's
baseline legs, never by the product package.

What it computes (§4.3, :305-333 and Eq. 9, :353-358; Appendix :1226,
:1262-1263), with the readings DESIGN.md R22-R28 lists where the paper is silent:
  gaussian_blur   G(I, sigma): separable normalised Gaussian, radius ceil(3 sigma),
                  reflect padding (R23)
  dog_mask        M_omega (Eq. 7): luminance of I_gt (R24), bilinear downsample by
                  0.2 (:1226, :1262), DoG = G(., 0.2 + 20 w) - G(., 0.1 + 10 w),
                  |.| min-max normalised (R25), > 0.5 (:318); for 0 <= w <= 0.5 the
                  complement 1 - M (:327); nearest-neighbour upsample (:1226)
  freq_loss       L_omega = ||(I - I_gt) . M_omega||_1 (Eq. 8), as a mean (R26)
  ssim            11 x 11 Gaussian window, sigma 1.5, C1 = 0.01^2, C2 = 0.03^2,
                  zero padding, mean over pixels and channels (R27; "kept the same"
                  as Gaussian splatting, :397)
  total_loss      L = l_L1 L1 + l_ssim (1 - SSIM) + l_w L_omega, l_ssim = 0.2,
                  l_w = 0.5, l_L1 = 1 - l_ssim - l_w (Eq. 9, :355-357, :1252-1263)
Every loss returns (value, dL/dI) with the gradient derived by hand.
Images are [3][H][W] float64 in [0, 1].
"""
from __future__ import annotations

import math

import numpy as np

LAMBDA_SSIM = 0.2
LAMBDA_OMEGA = 0.5
EPS_OMEGA = 0.5       # PAPER.md:318 "we pick 0.5"
DOWNSAMPLE = 0.2      # PAPER.md:1262 scale_im,freq
SSIM_WIN, SSIM_SIGMA = 11, 1.5
C1, C2 = 0.01 ** 2, 0.03 ** 2


def gaussian_kernel1d(sigma: float) -> np.ndarray:
    """Normalised taps exp(-i^2 / (2 sigma^2)), i in [-r, r], r = ceil(3 sigma); sigma = 0: [1]."""
    if sigma <= 0:
        return np.ones(1)
    r = int(math.ceil(3.0 * sigma))
    i = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-(i * i) / (2.0 * sigma * sigma))
    return w / w.sum()


def _reflect_index(i: np.ndarray, n: int) -> np.ndarray:
    """numpy/torch 'reflect' (mirror without repeating the edge), any distance."""
    if n == 1:
        return np.zeros_like(i)
    period = 2 * (n - 1)
    i = np.mod(i, period)
    return np.where(i < n, i, period - i)


def _conv1d(x: np.ndarray, w: np.ndarray, axis: int, pad: str) -> np.ndarray:
    """out[i] = sum_k w[k] x[i + k - r] along `axis`, out-of-range samples
    reflected ('reflect') or zero ('zero')."""
    r = (w.size - 1) // 2
    n = x.shape[axis]
    out = np.zeros_like(x, dtype=np.float64)
    idx = np.arange(n)
    for k in range(w.size):
        src = idx + k - r
        if pad == "reflect":
            out += w[k] * np.take(x, _reflect_index(src, n), axis=axis)
        else:
            ok = (src >= 0) & (src < n)
            sh = np.take(x, np.clip(src, 0, n - 1), axis=axis)
            m = ok.reshape([-1 if a == axis else 1 for a in range(x.ndim)])
            out += w[k] * np.where(m, sh, 0.0)
    return out


def gaussian_blur(img2d: np.ndarray, sigma: float) -> np.ndarray:
    """G(I, sigma) of PAPER.md:310 on one [H][W] plane (separable, reflect padding)."""
    w = gaussian_kernel1d(sigma)
    return _conv1d(_conv1d(np.asarray(img2d, np.float64), w, 1, "reflect"), w, 0, "reflect")


def luminance(img3: np.ndarray) -> np.ndarray:
    return 0.299 * img3[0] + 0.587 * img3[1] + 0.114 * img3[2]


def down_size(n: int, scale: float = DOWNSAMPLE) -> int:
    return max(1, int(math.floor(n * scale + 0.5)))


def downsample_bilinear(img2d: np.ndarray, scale: float = DOWNSAMPLE) -> np.ndarray:
    """Bilinear resample to (down_size(H), down_size(W)); output pixel centre i maps
    to source coordinate (i + 0.5) H / Hd - 0.5, clamped to the image."""
    H, W = img2d.shape
    Hd, Wd = down_size(H, scale), down_size(W, scale)

    def coords(n_out, n_in):
        c = (np.arange(n_out) + 0.5) * (n_in / n_out) - 0.5
        c = np.clip(c, 0.0, n_in - 1)
        i0 = np.floor(c).astype(np.int64)
        i1 = np.minimum(i0 + 1, n_in - 1)
        return i0, i1, c - i0

    y0, y1, fy = coords(Hd, H)
    x0, x1, fx = coords(Wd, W)
    a = img2d[y0][:, x0] * (1 - fx)[None, :] + img2d[y0][:, x1] * fx[None, :]
    b = img2d[y1][:, x0] * (1 - fx)[None, :] + img2d[y1][:, x1] * fx[None, :]
    return a * (1 - fy)[:, None] + b * fy[:, None]


def dog_response(gt3: np.ndarray, omega: float, scale: float = DOWNSAMPLE) -> np.ndarray:
    """|DoG_omega| of Eq. 7 on the downsampled luminance, min-max normalised to [0, 1]
    (a constant response maps to 0)."""
    lo = downsample_bilinear(luminance(np.asarray(gt3, np.float64)), scale)
    d = np.abs(gaussian_blur(lo, 0.2 + 20.0 * omega) - gaussian_blur(lo, 0.1 + 10.0 * omega))
    mn, mx = d.min(), d.max()
    return (d - mn) / (mx - mn) if mx > mn else np.zeros_like(d)


def dog_mask(gt3: np.ndarray, omega: float, eps: float = EPS_OMEGA, scale: float = DOWNSAMPLE) -> np.ndarray:
    """M_omega (Eq. 7) at the downsampled resolution, uint8 {0, 1}; complement for omega <= 0.5."""
    m = dog_response(gt3, omega, scale) > eps
    if omega <= 0.5:
        m = ~m
    return m.astype(np.uint8)


def upsample_nearest(mask_lo: np.ndarray, H: int, W: int) -> np.ndarray:
    """Full-resolution pixel (i, j) takes mask_lo[floor(i Hd / H), floor(j Wd / W)]."""
    Hd, Wd = mask_lo.shape
    iy = np.minimum((np.arange(H) * Hd) // H, Hd - 1)
    ix = np.minimum((np.arange(W) * Wd) // W, Wd - 1)
    return mask_lo[iy][:, ix]


def l1_loss(img, gt):
    d = np.asarray(img, np.float64) - np.asarray(gt, np.float64)
    n = d.size
    return float(np.abs(d).sum() / n), np.sign(d) / n


def freq_loss(img, gt, mask_full):
    """L_omega = mean over pixels and channels of |I - I_gt| M (Eq. 8, R26)."""
    d = np.asarray(img, np.float64) - np.asarray(gt, np.float64)
    m = np.asarray(mask_full, np.float64)[None]
    n = d.size
    return float((np.abs(d) * m).sum() / n), np.sign(d) * m / n


def ssim_window() -> np.ndarray:
    i = np.arange(SSIM_WIN, dtype=np.float64) - SSIM_WIN // 2
    w = np.exp(-(i * i) / (2.0 * SSIM_SIGMA ** 2))
    return w / w.sum()


def _blur_zero(x):
    w = ssim_window()
    return _conv1d(_conv1d(x, w, 1, "zero"), w, 0, "zero")


def ssim_map(xc, yc):
    """Per-pixel SSIM of one channel (the map whose mean is SSIM)."""
    mx, my = _blur_zero(xc), _blur_zero(yc)
    exx, eyy, exy = _blur_zero(xc * xc), _blur_zero(yc * yc), _blur_zero(xc * yc)
    return ((2 * mx * my + C1) * (2 * (exy - mx * my) + C2) /
            ((mx * mx + my * my + C1) * ((exx - mx * mx) + (eyy - my * my) + C2)))


def ssim(img, gt):
    """Mean SSIM over pixels and channels and d mean SSIM / d img (R27).
    Per channel: mu = G*x, E2 = G*x^2, Exy = G*(x y) (zero padding),
    S = (2 mu_x mu_y + C1)(2 (Exy - mu_x mu_y) + C2) /
        ((mu_x^2 + mu_y^2 + C1)((E2x - mu_x^2) + (E2y - mu_y^2) + C2));
    dS/dmu_x = (2 mu_y A2 - 2 mu_y A1) / (B1 B2) - S (2 mu_x / B1 - 2 mu_x / B2),
    dS/dE2x = -S / B2, dS/dExy = 2 A1 / (B1 B2); the window's adjoint (the same
    symmetric zero-padded blur) carries them back to the pixels:
    d mean S / dx = (G*d_mu + 2 x G*d_E2 + y G*d_Exy) / N."""
    x = np.asarray(img, np.float64)
    y = np.asarray(gt, np.float64)
    N = x.size
    total = 0.0
    grad = np.zeros_like(x)
    for c in range(x.shape[0]):
        xc, yc = x[c], y[c]
        mx, my = _blur_zero(xc), _blur_zero(yc)
        exx, eyy, exy = _blur_zero(xc * xc), _blur_zero(yc * yc), _blur_zero(xc * yc)
        A1 = 2 * mx * my + C1
        A2 = 2 * (exy - mx * my) + C2
        B1 = mx * mx + my * my + C1
        B2 = (exx - mx * mx) + (eyy - my * my) + C2
        S = A1 * A2 / (B1 * B2)
        total += S.sum()
        d_mu = (2 * my * A2 - 2 * my * A1) / (B1 * B2) - S * (2 * mx / B1 - 2 * mx / B2)
        d_e2 = -S / B2
        d_exy = 2 * A1 / (B1 * B2)
        grad[c] = (_blur_zero(d_mu) + 2 * xc * _blur_zero(d_e2) + yc * _blur_zero(d_exy)) / N
    return float(total / N), grad


def total_loss(img, gt, mask_full, lambda_ssim: float = LAMBDA_SSIM, lambda_omega: float = LAMBDA_OMEGA):
    """Eq. 9: (L, dL/dI, parts) with L = l_L1 L1 + l_ssim (1 - SSIM) + l_w L_omega."""
    l1, g1 = l1_loss(img, gt)
    s, gs = ssim(img, gt)
    lw, gw = freq_loss(img, gt, mask_full)
    lam_l1 = 1.0 - lambda_ssim - lambda_omega
    L = lam_l1 * l1 + lambda_ssim * (1.0 - s) + lambda_omega * lw
    g = lam_l1 * g1 - lambda_ssim * gs + lambda_omega * gw
    return L, g, {"l1": l1, "ssim": s, "freq": lw}


def omega_schedule(iteration: int, total_iterations: int) -> float:
    """The linear schedule omega = current / total."""
    return float(iteration) / float(total_iterations)
