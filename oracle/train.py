"""Plain fp64 numpy oracle of the optimizer and shape-aware density control
(SURVEY.md §8(f) NEXT-2).  TEST INFRASTRUCTURE ONLY.

PAPER.md §4.4 (:348-358) and Appendix (:1227-1271), with the readings DESIGN.md
R29-R33 lists where the paper is silent or conflicting:
  adam_step        Adam with bias correction (beta1 0.9, beta2 0.999, eps 1e-15),
                   per-group learning rates (:1231-1244); SH DC takes lr_feature,
                   the higher bands lr_feature / 20 (R29)
  lr_position      log-linear decay 1.6e-4 -> 1.6e-6 over 30000 steps with the delay
                   multiplier 0.01 (:1232-1236; delay_steps = 0 -> no warm-up, R29)
  reset_opacity    kappa <- min(kappa, 0.01) (R30)        reset_shape   beta <- 2 (R30)
  densify_prune    per particle: prune if kappa < 0.005 or phi-bar(beta) < 0.5 (R31);
                   else, if the mean view-space gradient norm >= 3e-4 (:1250): clone
                   when max exp(log s) <= 0.01 x extent, otherwise split into two
                   children with scales / 1.6 at mu + R (s . z), z ~ N(0, I) from the
                   shared counter-based generator (R32); kept particles keep their
                   Adam moments, clones and both split children start at zero (R33);
                   order: [kept / cloned originals / first split children in index
                   order], then [clones], then [second split children] (R33)
The normal draws come from `normal3` below -- splitmix64 on (seed, particle,
child) and Box-Muller -- which the CUDA path implements independently.
Parameters are the planar [C][P] layout (mean 3, log_scale 3, quat 4,
opacity_logit 1, sh 3K, beta 1).
"""
from __future__ import annotations

import math

import numpy as np

BETA1, BETA2, ADAM_EPS = 0.9, 0.999, 1e-15
LR = {"pos_init": 1.6e-4, "pos_final": 1.6e-6, "pos_delay_mult": 0.01, "pos_max_steps": 30000,
      "feature": 2.5e-3, "opacity": 0.05, "scaling": 5e-3, "rotation": 1e-3, "shape": 1e-3}
OPACITY_PRUNE, SHAPE_PRUNE, DENSIFY_GRAD, PERCENT_DENSE, SPLIT_DIV = 0.005, 0.5, 3e-4, 0.01, 1.6
OPACITY_RESET = 0.01


def plane_groups(K: int):
    """(name, first plane, plane count) of the planar parameter layout."""
    return [("mean", 0, 3), ("log_scale", 3, 3), ("quat", 6, 4), ("opacity_logit", 10, 1),
            ("sh", 11, 3 * K), ("beta", 11 + 3 * K, 1)]


def lr_position(step: int, init=LR["pos_init"], final=LR["pos_final"], delay_mult=LR["pos_delay_mult"],
                max_steps=LR["pos_max_steps"], delay_steps=0) -> float:
    """Log-linear interpolation init -> final over max_steps; the delay multiplier
    ramps the rate in over delay_steps (none with the default 0)."""
    if step < 0 or (init == 0.0 and final == 0.0):
        return 0.0
    if delay_steps > 0:
        delay = delay_mult + (1 - delay_mult) * math.sin(0.5 * math.pi * min(max(step / delay_steps, 0.0), 1.0))
    else:
        delay = 1.0
    t = min(max(step / max_steps, 0.0), 1.0)
    return delay * math.exp(math.log(init) * (1 - t) + math.log(final) * t)


def plane_lrs(K: int, step: int) -> np.ndarray:
    lr = np.zeros(3 + 3 + 4 + 1 + 3 * K + 1)
    lr[0:3] = lr_position(step)
    lr[3:6] = LR["scaling"]
    lr[6:10] = LR["rotation"]
    lr[10] = LR["opacity"]
    lr[11:14] = LR["feature"]                 # SH DC (planes 3k + c, k = 0)
    lr[14:11 + 3 * K] = LR["feature"] / 20.0  # higher bands
    lr[11 + 3 * K] = LR["shape"]
    return lr


def adam_step(params, grads, m, v, step: int, K: int):
    """One bias-corrected Adam step (step >= 1), planar [C][P] arrays, in place copies returned."""
    lr = plane_lrs(K, step)[:, None]
    m2 = BETA1 * m + (1 - BETA1) * grads
    v2 = BETA2 * v + (1 - BETA2) * grads * grads
    mh = m2 / (1 - BETA1 ** step)
    vh = v2 / (1 - BETA2 ** step)
    return params - lr * mh / (np.sqrt(vh) + ADAM_EPS), m2, v2


def _logit(p):
    return math.log(p / (1 - p))


def reset_opacity(params, K: int):
    out = params.copy()
    cap = _logit(OPACITY_RESET)
    out[10] = np.minimum(out[10], cap)
    return out


def reset_shape(params, K: int):
    out = params.copy()
    out[11 + 3 * K] = 2.0
    return out


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def uniform24(seed: int, particle: int, child: int, k: int) -> float:
    """u in (0, 1): the top 24 bits of splitmix64(seed, particle, child, k), + 0.5, / 2^24."""
    key = (seed * 0x100000001B3 + particle * 16 + child * 4 + k) & 0xFFFFFFFFFFFFFFFF
    return ((_splitmix64(key) >> 40) + 0.5) / 16777216.0


def normal3(seed: int, particle: int, child: int) -> np.ndarray:
    """Three N(0, 1) draws: Box-Muller on uniform24 k = 0, 1 (two normals) and 2, 3 (one)."""
    u0, u1, u2, u3 = (uniform24(seed, particle, child, k) for k in range(4))
    r0, r1 = math.sqrt(-2.0 * math.log(u0)), math.sqrt(-2.0 * math.log(u2))
    return np.array([r0 * math.cos(2 * math.pi * u1), r0 * math.sin(2 * math.pi * u1), r1 * math.cos(2 * math.pi * u3)])


def quat_to_rot(q):
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def phi_bar(beta, rho):
    return 2.0 / (1.0 + np.exp(-rho * (np.asarray(beta, np.float64) - 2.0)))


def densify_actions(params, grad_accum, grad_count, K: int, extent: float, rho: float):
    """Per particle: 0 prune, 1 keep, 2 clone, 3 split (R31, R32)."""
    kappa = 1.0 / (1.0 + np.exp(-params[10]))
    phib = phi_bar(params[11 + 3 * K], rho)
    smax = np.exp(params[3:6]).max(axis=0)
    avg = np.where(grad_count > 0, grad_accum / np.maximum(grad_count, 1), 0.0)
    act = np.ones(params.shape[1], np.int32)
    dens = avg >= DENSIFY_GRAD
    act[dens & (smax <= PERCENT_DENSE * extent)] = 2
    act[dens & (smax > PERCENT_DENSE * extent)] = 3
    act[(kappa < OPACITY_PRUNE) | (phib < SHAPE_PRUNE)] = 0
    return act


def densify_prune(params, m, v, grad_accum, grad_count, K: int, extent: float, rho: float, seed: int):
    """The new particle set (R33 order): every non-pruned particle in index order
    (split parents become their first child), then the clones, then the second
    split children.  Returns (params', m', v', actions)."""
    act = densify_actions(params, grad_accum, grad_count, K, extent, rho)
    P = params.shape[1]
    keep = np.nonzero(act > 0)[0]
    clones = np.nonzero(act == 2)[0]
    splits = np.nonzero(act == 3)[0]
    out = [params[:, keep].copy()]
    mo, vo = [m[:, keep].copy()], [v[:, keep].copy()]
    # split parents (in place, first child) and the second children
    pos = {int(i): j for j, i in enumerate(keep)}
    second = np.zeros((params.shape[0], splits.size))
    for c, i in enumerate(splits):
        R = quat_to_rot(params[6:10, i])
        s = np.exp(params[3:6, i])
        for child in (0, 1):
            p = params[:, i].copy()
            p[0:3] = params[0:3, i] + R @ (s * normal3(seed, int(i), child))
            p[3:6] = params[3:6, i] - math.log(SPLIT_DIV)
            if child == 0:
                out[0][:, pos[int(i)]] = p
                mo[0][:, pos[int(i)]] = 0.0
                vo[0][:, pos[int(i)]] = 0.0
            else:
                second[:, c] = p
    out += [params[:, clones].copy(), second]
    mo += [np.zeros((m.shape[0], clones.size)), np.zeros_like(second)]
    vo += [np.zeros((v.shape[0], clones.size)), np.zeros_like(second)]
    assert P >= 0
    return np.concatenate(out, axis=1), np.concatenate(mo, axis=1), np.concatenate(vo, axis=1), act


def viewspace_grad_norm(du, dv, W: int, H: int):
    """The densification statistic per view: |dL/d(ndc)| = |(du W/2, dv H/2)| (R32)."""
    return np.sqrt((du * 0.5 * W) ** 2 + (dv * 0.5 * H) ** 2)
