"""GPU parity of the loss front end against oracle/loss.py.

Bars: the mask M_omega equal to the oracle's except at pixels whose normalised
|DoG| lies within 1e-3 of eps_omega (fp32 blurs vs fp64: the decision is
ambiguous there, R18 applied to Eq. 7), which must be rare; L1 and
L_omega within 2e-6 absolute, SSIM and the total within 2e-5 (fp32 variance
cancellation); dL/dimage within 1e-3 relative plus 1e-3 of its largest entry
(plus the L1/L_omega subgradients' sign agreement).  Sizes: ragged tiles, and
BASELINE config 3 (1297 x 840) in full.
"""
import numpy as np
import pytest
import torch

import paper_2402_10128_b200 as G
from oracle import loss as LO

pytestmark = pytest.mark.gpu


def smooth_image(H, W, seed):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    img = np.zeros((3, H, W))
    for _ in range(12):
        cy, cx = rng.uniform(0, H), rng.uniform(0, W)
        s = rng.uniform(3, 0.2 * max(H, W))
        amp = rng.uniform(-0.5, 0.5, 3)
        g = np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * s * s))
        img += amp[:, None, None] * g[None]
    img += 0.02 * rng.normal(size=img.shape)
    img[:, :, W // 3:W // 3 + 2] += 0.4   # a sharp edge
    return np.clip(img + 0.5, 0, 1).astype(np.float32)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("H,W", [(120, 200), (97, 131), (840, 1297)])
@pytest.mark.parametrize("omega", [0.0, 0.25, 0.5, 0.6, 0.9, 1.0])
def test_mask_parity(H, W, omega):
    gt = smooth_image(H, W, 7)
    loss = G.Loss(W, H)
    m = loss.mask(dev(gt), omega).cpu().numpy()
    ref = LO.dog_mask(gt.astype(np.float64), omega)
    assert m.shape == ref.shape == (LO.down_size(H), LO.down_size(W))
    resp = LO.dog_response(gt.astype(np.float64), omega)
    amb = np.abs(resp - 0.5) < 1e-3
    assert amb.mean() < 0.01
    bad = (m != ref) & ~amb
    assert not bad.any(), (int(bad.sum()), np.argwhere(bad)[:5])


@pytest.mark.parametrize("H,W", [(64, 96), (97, 131), (840, 1297)])
def test_loss_value_and_gradient_parity(H, W):
    rng = np.random.default_rng(H + W)
    gt = smooth_image(H, W, 3)
    img = np.clip(gt + rng.normal(0, 0.1, gt.shape).astype(np.float32), 0, 1)
    mask_lo = LO.dog_mask(gt.astype(np.float64), 0.7)
    loss = G.Loss(W, H)
    out, g = loss(dev(img), dev(gt), dev(mask_lo))
    torch.cuda.synchronize()
    out, g = out.cpu().numpy().astype(np.float64), g.cpu().numpy().astype(np.float64)
    mfull = LO.upsample_nearest(mask_lo, H, W)
    L, gref, parts = LO.total_loss(img.astype(np.float64), gt.astype(np.float64), mfull)
    # L1 / L_omega: fp32 sums of exact terms; SSIM: fp32 variances E[x^2] - mu^2 cancel
    # (relative error ~1e-7 E[x^2] / var per pixel), hence 2e-5 on the mean map
    ref = np.array([L, parts["l1"], parts["ssim"], parts["freq"]])
    assert np.all(np.abs(out - ref) <= np.array([2e-5, 2e-6, 2e-5, 2e-6])), (out, ref)
    # the north_star's gradient bar, 1e-3 relative, with a floor of 1e-3 of the largest
    # entry for the few pixels whose SSIM terms cancel
    assert np.all(np.abs(g - gref) <= 1e-3 * np.abs(gref) + 1e-3 * np.abs(gref).max())


def test_loss_without_mask_and_identity():
    H, W = 50, 70
    gt = smooth_image(H, W, 9)
    loss = G.Loss(W, H)
    out, g = loss(dev(gt), dev(gt), None)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert abs(o[0]) < 1e-6 and o[1] == 0.0 and abs(o[2] - 1.0) < 1e-6 and o[3] == 0.0
    assert np.abs(g.cpu().numpy()).max() < 1e-7    # rounding-level vs the 1/N ~ 1e-4 scale of dL/dI


def test_training_step_composes_render_loss_backward():
    """render -> Eq. 9 loss -> dL/dimage -> ges_render_bwd: the gradient the
    rasterizer receives is the loss kernels' output (one real training step)."""
    import ges_inputs as gi
    sc = gi.make_config(0, P=1500)
    cam = sc.cameras[0]
    params = G.PlanarParams.from_inputs(sc.particles)
    r = G.Renderer(params.P, cam.width, cam.height)
    st = G.Settings(rho=0.1)
    gt = dev(smooth_image(cam.height, cam.width, 4))
    loss = G.Loss(cam.width, cam.height)
    mask = loss.mask(gt, 0.3)
    img = r.forward(params, cam, st)
    out, dL = loss(img, gt, mask)
    grads = r.backward(params, cam, st, dL)
    torch.cuda.synchronize()
    assert np.isfinite(out.cpu().numpy()).all() and out[0].item() > 0
    assert all(torch.isfinite(getattr(grads, n)).all() for n in G.PARAM_NAMES)
    assert grads.mean.abs().sum().item() > 0
