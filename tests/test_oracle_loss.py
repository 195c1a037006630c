"""Pins of the loss-front-end oracle (oracle/loss.py).

Checked against what the mathematics fixes, not against the oracle itself:
  * blur: an interior impulse becomes the closed-form normalised Gaussian
    outer product; sigma = 0 is the identity; constants are invariant; the
    reflect padding equals numpy's 'reflect' convention
  * bilinear downsample reproduces an affine ramp exactly (interior)
  * DoG mask (Eq. 7): a constant image has zero response (mask 0 for
    omega > 0.5, its complement 1 below); the complement rule of PAPER.md:327;
    a step edge is found only along the edge at a high-frequency omega
  * SSIM: 1 for identical images with zero gradient; the closed form
    (2ab + C1)/(a^2 + b^2 + C1) for constant images away from the border
  * every loss gradient (L1, L_omega, SSIM, Eq. 9's total) against central
    finite differences; Eq. 9's weights (0.3, 0.2, 0.5)
"""
import math

import numpy as np
import pytest

from oracle import loss as LO


def test_blur_impulse_closed_form_identity_and_constant():
    img = np.zeros((41, 45))
    img[20, 22] = 1.0
    for sigma in (0.7, 1.5, 3.2):
        out = LO.gaussian_blur(img, sigma)
        r = math.ceil(3 * sigma)
        z = sum(math.exp(-i * i / (2 * sigma * sigma)) for i in range(-r, r + 1))
        for (dy, dx) in ((0, 0), (1, 0), (2, -3), (r, r), (-r, 1)):
            expect = math.exp(-(dx * dx + dy * dy) / (2 * sigma * sigma)) / (z * z)
            assert abs(out[20 + dy, 22 + dx] - expect) < 1e-15
        assert abs(out[20 + r + 1, 22]) == 0.0
        assert abs(out.sum() - 1.0) < 1e-12
    assert np.array_equal(LO.gaussian_blur(img, 0.0), img)
    c = np.full((9, 13), 0.37)
    assert np.allclose(LO.gaussian_blur(c, 2.5), c, rtol=0, atol=1e-15)


def test_reflect_padding_convention():
    x = np.arange(7.0)
    for n_pad in (3, 6, 13):
        idx = LO._reflect_index(np.arange(-n_pad, 7 + n_pad), 7)
        assert np.array_equal(x[idx], np.pad(x, n_pad, mode="reflect"))


def test_bilinear_downsample_affine_and_constant():
    H, W = 50, 65
    yy, xx = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    ramp = 0.3 + 0.01 * xx - 0.02 * yy
    lo = LO.downsample_bilinear(ramp, 0.2)
    Hd, Wd = LO.down_size(H), LO.down_size(W)
    assert lo.shape == (Hd, Wd) == (10, 13)
    cy = (np.arange(Hd) + 0.5) * H / Hd - 0.5
    cx = (np.arange(Wd) + 0.5) * W / Wd - 0.5
    assert np.allclose(lo, 0.3 + 0.01 * cx[None, :] - 0.02 * cy[:, None], rtol=0, atol=1e-13)
    assert np.allclose(LO.downsample_bilinear(np.full((H, W), 0.6)), 0.6, rtol=0, atol=1e-15)


def test_dog_mask_constant_complement_and_edge():
    H, W = 80, 120
    const = np.full((3, H, W), 0.4)
    for om in (0.6, 0.75, 1.0):
        assert not LO.dog_mask(const, om).any()
    for om in (0.0, 0.2, 0.5):
        assert LO.dog_mask(const, om).all()
    rng = np.random.default_rng(3)
    img = rng.uniform(0, 1, (3, H, W))
    for om in (0.1, 0.3, 0.45):
        raw = (LO.dog_response(img, om) > 0.5).astype(np.uint8)
        assert np.array_equal(LO.dog_mask(img, om), 1 - raw)
    # a vertical step edge: the band-pass response is odd about the edge (0 on it),
    # peaks within ~sigma of it and vanishes far away -> two bands around the edge
    step = np.zeros((3, 400, 600))
    step[:, :, 300:] = 1.0
    m = LO.dog_mask(step, 0.55)      # sigma2 = 5.6, sigma1 = 11.2 (downsampled px)
    Wd = m.shape[1]
    cols = np.nonzero(m.any(axis=0))[0]
    assert cols.size > 0 and np.all(m[:, cols].all(axis=0))   # full-height bands
    assert abs(cols.mean() - (Wd / 2 - 0.5)) < 1.0            # symmetric about the edge
    assert cols.min() > Wd / 2 - 25 and cols.max() < Wd / 2 + 25
    assert m[:, :10].sum() == 0 and m[:, -10:].sum() == 0


def test_ssim_identity_and_constant_closed_form():
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (3, 20, 24))
    s, g = LO.ssim(x, x)
    assert abs(s - 1.0) < 1e-12
    assert np.abs(g).max() < 1e-12
    a, b = 0.3, 0.8
    m = LO.ssim_map(np.full((30, 30), a), np.full((30, 30), b))
    expect = (2 * a * b + LO.C1) / (a * a + b * b + LO.C1)
    assert np.allclose(m[5:25, 5:25], expect, rtol=0, atol=1e-11)   # var = E[x^2] - mu^2 rounds to ~1e-17


def _fd(f, x, idx_list, h=1e-6):
    out = []
    for idx in idx_list:
        xp = x.copy(); xp[idx] += h
        xm = x.copy(); xm[idx] -= h
        out.append((f(xp) - f(xm)) / (2 * h))
    return np.array(out)


@pytest.mark.parametrize("which", ["l1", "freq", "ssim", "total"])
def test_loss_gradients_finite_differences(which):
    rng = np.random.default_rng(11)
    H, W = 12, 10
    gt = rng.uniform(0, 1, (3, H, W))
    img = np.clip(gt + rng.normal(0, 0.2, gt.shape), 0, 1)
    img[np.abs(img - gt) < 1e-3] += 0.01       # stay off the |.| kink
    mask = (rng.uniform(0, 1, (H, W)) > 0.4).astype(np.uint8)
    fns = {"l1": lambda x: LO.l1_loss(x, gt), "freq": lambda x: LO.freq_loss(x, gt, mask),
           "ssim": lambda x: LO.ssim(x, gt), "total": lambda x: LO.total_loss(x, gt, mask)[:2]}
    f = fns[which]
    _, g = f(img)
    idx = [tuple(rng.integers(0, s) for s in img.shape) for _ in range(40)]
    fd = _fd(lambda x: f(x)[0], img, idx)
    an = np.array([g[i] for i in idx])
    assert np.allclose(an, fd, rtol=1e-5, atol=1e-10), np.abs(an - fd).max()


def test_total_loss_weights_and_zero_at_gt():
    assert abs((1 - LO.LAMBDA_SSIM - LO.LAMBDA_OMEGA) - 0.3) < 1e-15
    rng = np.random.default_rng(2)
    gt = rng.uniform(0, 1, (3, 16, 16))
    L, g, parts = LO.total_loss(gt, gt, np.ones((16, 16), np.uint8))
    assert abs(L) < 1e-12 and parts["l1"] == 0.0 and parts["freq"] == 0.0
    assert LO.omega_schedule(0, 40000) == 0.0 and LO.omega_schedule(20000, 40000) == 0.5


def test_upsample_nearest_covers_and_repeats():
    lo = np.arange(12, dtype=np.uint8).reshape(3, 4)
    up = LO.upsample_nearest(lo, 15, 20)
    assert up.shape == (15, 20)
    assert np.array_equal(up[::5, ::5], lo)
    assert np.array_equal(up[4, 4], lo[0, 0]) and np.array_equal(up[5, 5], lo[1, 1])
