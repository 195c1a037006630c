"""Pins of the optimizer / density-control oracle (oracle/train.py).

  * Adam: the first step from zero moments is -lr sign(g) per plane group; under a
    constant gradient every bias-corrected step is -lr sign(g) again (closed forms)
  * the position schedule's endpoints and its geometric midpoint (log-linear)
  * resets: kappa capped at exactly 0.01, beta = 2 (phi-bar = 1), both idempotent
  * densify/prune decisions on constructed particles (each action), counts and
    order of the new set, split children scales = parent / 1.6 and positions that
    reconstruct the generator's draws exactly; the generator's N(0, 1) moments
"""
import math

import numpy as np

from oracle import train as TR


def planar(P, K, rng):
    C = 3 + 3 + 4 + 1 + 3 * K + 1
    p = rng.normal(0, 1, (C, P))
    p[3:6] = rng.normal(-3, 0.3, (3, P))
    p[11 + 3 * K] = rng.uniform(0.5, 4, P)
    return p


def test_adam_first_and_constant_gradient_steps():
    rng = np.random.default_rng(0)
    K, P = 4, 7
    p = planar(P, K, rng)
    g = rng.normal(0, 1e-3, p.shape)
    m = np.zeros_like(p); v = np.zeros_like(p)
    lr = TR.plane_lrs(K, 1)[:, None]
    p1, m1, v1 = TR.adam_step(p, g, m, v, 1, K)
    assert np.allclose(p1 - p, -lr * np.sign(g), rtol=1e-9, atol=0)
    pp, mm, vv = p, m, v
    for step in range(1, 6):
        pn, mm, vv = TR.adam_step(pp, g, mm, vv, step, K)
        assert np.allclose(pn - pp, -TR.plane_lrs(K, step)[:, None] * np.sign(g), rtol=1e-9, atol=0)
        pp = pn
    lrs = TR.plane_lrs(K, 0)
    assert lrs[0] == TR.LR["pos_init"] and lrs[11] == TR.LR["feature"] and lrs[14] == TR.LR["feature"] / 20
    assert lrs[10] == 0.05 and lrs[3] == 0.005 and lrs[6] == 0.001 and lrs[-1] == 0.001


def test_position_schedule():
    assert TR.lr_position(0) == 1.6e-4
    assert abs(TR.lr_position(30000) - 1.6e-6) < 1e-18 and TR.lr_position(40000) == TR.lr_position(30000)
    assert abs(TR.lr_position(15000) - math.sqrt(1.6e-4 * 1.6e-6)) < 1e-15
    assert TR.lr_position(100, delay_steps=1000) < TR.lr_position(100)


def test_resets():
    rng = np.random.default_rng(1)
    K = 1
    p = planar(20, K, rng)
    p[10, :5] = 5.0
    r = TR.reset_opacity(p, K)
    kap = 1 / (1 + np.exp(-r[10]))
    assert np.all(kap <= 0.01 + 1e-15) and np.allclose(kap[:5], 0.01, rtol=1e-12)
    small = p[10] < math.log(0.01 / 0.99)
    assert np.array_equal(r[10][small], p[10][small])
    assert np.array_equal(TR.reset_opacity(r, K), r)
    s = TR.reset_shape(p, K)
    assert np.all(s[11 + 3 * K] == 2.0) and np.all(TR.phi_bar(s[11 + 3 * K], 0.1) == 1.0)
    assert np.array_equal(TR.reset_shape(s, K), s)


def test_densify_actions_and_new_set():
    rng = np.random.default_rng(2)
    K, P, extent = 1, 8, 10.0
    p = planar(P, K, rng)
    p[10] = 2.0                              # kappa 0.88
    p[3:6] = math.log(0.05)                   # max scale 0.05 <= 0.01 x 10 -> clone size
    p[11 + 3 * K] = 2.0
    acc = np.zeros(P); cnt = np.ones(P)
    acc[[1, 4]] = 1e-3                        # over the 3e-4 threshold
    p[3:6, 4] = math.log(0.5)                 # large -> split
    p[10, 2] = -7.0                           # kappa 9e-4 -> prune
    p[11 + 3 * K, 6] = -20.0                  # phi-bar(-20) = 0.2 < 0.5 -> prune
    act = TR.densify_actions(p, acc, cnt, K, extent, 0.1)
    assert list(act) == [1, 2, 0, 1, 3, 1, 0, 1]
    m = rng.normal(0, 1, p.shape); v = np.abs(rng.normal(0, 1, p.shape))
    q, mq, vq, _ = TR.densify_prune(p, m, v, acc, cnt, K, extent, 0.1, seed=7)
    assert q.shape[1] == P - 2 + 1 + 1
    kept = [0, 1, 3, 4, 5, 7]
    for j, i in enumerate(kept):
        if i != 4:
            assert np.array_equal(q[:, j], p[:, i]) and np.array_equal(mq[:, j], m[:, i])
    assert np.array_equal(q[:, 6], p[:, 1]) and not mq[:, 6].any()          # the clone
    R = TR.quat_to_rot(p[6:10, 4])
    s = np.exp(p[3:6, 4])
    for col, child in ((3, 0), (7, 1)):                                     # the split children
        assert np.allclose(q[3:6, col], p[3:6, 4] - math.log(1.6), rtol=0, atol=1e-15)
        z = (R.T @ (q[0:3, col] - p[0:3, 4])) / s
        assert np.allclose(z, TR.normal3(7, 4, child), rtol=0, atol=1e-12)
        assert not mq[:, col].any() and not vq[:, col].any()
        assert np.array_equal(q[6:, col][5:], p[6:, 4][5:])


def test_generator_moments_and_viewspace_norm():
    z = np.array([TR.normal3(3, i, c) for i in range(4000) for c in (0, 1)]).reshape(-1)
    assert abs(z.mean()) < 0.03 and abs(z.var() - 1) < 0.05
    u = np.array([TR.uniform24(1, i, 0, 0) for i in range(5000)])
    assert u.min() > 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.02
    assert abs(TR.viewspace_grad_norm(2e-6, 0.0, 800, 600) - 8e-4) < 1e-15
