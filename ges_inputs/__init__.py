"""Seeded synthetic inputs for the GES rasterizer (configs 0-4 of BASELINE.json).

This module is shared by the oracle tests and the CUDA path.  It holds NO part of
the method's arithmetic (no projection, no phi, no compositing): it only draws
random particles, builds pinhole cameras (a look-at pose is input construction,
not the method) and draws upstream image gradients.  numpy only.

Recipe:
  * all draws use ``numpy.random.default_rng(seed)``, seed = 1000 + config index;
    the upstream gradient of view v uses seed*100 + v;
  * particles are emitted planar SoA, float32, in the ABI order
    mean[3][P], log_scale[3][P], quat[4][P] (w,x,y,z), opacity_logit[P],
    sh[3K][P] (plane = 3*k + channel), beta[P] (the TRUE beta; the paper stores
    beta-2, which is only a storage shift).
The paper measured on Mip-NeRF360 / Tanks&Temples / Deep Blending;
none of those are available, so these seeded scenes of the same scale stand in.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

__all__ = [
    "Particles", "Camera", "Scene", "make_config", "look_at", "upstream_grad",
    "CONFIG_NAMES", "random_small_scene",
]

CONFIG_NAMES = {
    0: "cfg0_tiny_2k_256",
    1: "cfg1_beta_sweep_50k_512",
    2: "cfg2_object_300k_800_8views",
    3: "cfg3_unbounded_1p5M_1297x840",
    4: "cfg4_large_3M_1600x1064_64views",
}


@dataclasses.dataclass
class Particles:
    """Planar SoA particle parameters, float32."""
    mean: np.ndarray           # [3, P]
    log_scale: np.ndarray      # [3, P]
    quat: np.ndarray           # [4, P] (w, x, y, z)
    opacity_logit: np.ndarray  # [P]
    sh: np.ndarray             # [3K, P], plane 3*k + c
    beta: np.ndarray           # [P]
    sh_degree: int

    @property
    def P(self) -> int:
        return int(self.mean.shape[1])

    @property
    def K(self) -> int:
        return (self.sh_degree + 1) ** 2

    def planes(self):
        return [self.mean, self.log_scale, self.quat, self.opacity_logit[None, :],
                self.sh, self.beta[None, :]]

    def n_planes(self) -> int:
        return 3 + 3 + 4 + 1 + 3 * self.K + 1

    def flat(self) -> np.ndarray:
        """All planes stacked in ABI order as one contiguous [C][P] float32 array."""
        return np.ascontiguousarray(np.concatenate(self.planes(), axis=0), dtype=np.float32)

    def subset(self, idx) -> "Particles":
        return Particles(self.mean[:, idx].copy(), self.log_scale[:, idx].copy(),
                         self.quat[:, idx].copy(), self.opacity_logit[idx].copy(),
                         self.sh[:, idx].copy(), self.beta[idx].copy(), self.sh_degree)


@dataclasses.dataclass
class Camera:
    """Pinhole camera, world->camera rotation R (row-major 3x3) and translation t
    (OpenCV axes: x right, y down, z forward)."""
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    near: float
    R: np.ndarray  # [3,3] float32
    t: np.ndarray  # [3] float32


@dataclasses.dataclass
class Scene:
    name: str
    particles: Particles
    cameras: List[Camera]
    rho: float = 0.1
    background: tuple = (0.0, 0.0, 0.0)
    seed: int = 0


def look_at(center, target=(0.0, 0.0, 0.0), up=(0.0, -1.0, 0.0)):
    """World->camera (R, t) for a camera at `center` looking at `target` with world
    up `up` (OpenCV axes: rows of R are right, down, forward)."""
    c = np.asarray(center, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - c
    f /= np.linalg.norm(f)
    upv = np.asarray(up, dtype=np.float64)
    r = np.cross(f, upv)
    if np.linalg.norm(r) < 1e-6:  # looking along `up`: pick another reference
        r = np.cross(f, np.array([0.0, 0.0, 1.0]))
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f], axis=0)
    t = -R @ c
    return R.astype(np.float32), t.astype(np.float32)


def _camera(W, H, f, R, t, near=0.2):
    return Camera(int(W), int(H), float(np.float32(f)), float(np.float32(f)),
                  float(np.float32(W / 2.0)), float(np.float32(H / 2.0)), float(np.float32(near)),
                  np.asarray(R, np.float32).reshape(3, 3), np.asarray(t, np.float32).reshape(3))


def _quats(rng, P):
    q = rng.standard_normal((4, P))
    q /= np.linalg.norm(q, axis=0, keepdims=True)
    return q


def _sh3(rng, P, dc_sigma=0.5, hi_sigma=0.05):
    K = 16
    sh = rng.normal(0.0, hi_sigma, size=(3 * K, P))
    sh[0:3] = rng.normal(0.0, dc_sigma, size=(3, P))
    return sh


def _blob_and_shell(rng, P):
    n_blob = int(round(0.8 * P))
    n_shell = P - n_blob
    blob = rng.normal(0.0, 2.0, size=(3, n_blob))
    d = rng.standard_normal((3, n_shell))
    d /= np.linalg.norm(d, axis=0, keepdims=True)
    rad = rng.uniform(28.0, 30.0, size=n_shell)
    shell = d * rad
    mean = np.concatenate([blob, shell], axis=1)
    perm = rng.permutation(P)
    return mean[:, perm]


def _pack(mean, log_scale, quat, logit, sh, beta, deg) -> Particles:
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return Particles(f(mean), f(log_scale), f(quat), f(logit), f(sh), f(beta), deg)


def make_config(cfg: int, beta_value: Optional[float] = None, P: Optional[int] = None,
                n_views: Optional[int] = None) -> Scene:
    """Scene of BASELINE.json config `cfg` (0-4).  `P` overrides the particle count
    (same distributions), `beta_value` fixes beta (config 1's sweep), `n_views`
    truncates the camera list."""
    seed = 1000 + cfg
    rng = np.random.default_rng(seed)
    if cfg in (0, 1):
        P = P or (2000 if cfg == 0 else 50000)
        mean = rng.standard_normal((3, P)) + np.array([[0.0], [0.0], [4.0]])
        log_scale = rng.normal(-3.0, 0.5, size=(3, P))
        quat = _quats(rng, P)
        logit = rng.normal(0.0, 1.0, size=P)
        beta = rng.uniform(0.5, 4.0, size=P)
        if beta_value is not None:
            beta = np.full(P, beta_value)
        sh = rng.normal(0.0, 0.3, size=(3, P))
        W = H = 256 if cfg == 0 else 512
        f = 300.0 if cfg == 0 else 600.0
        cams = [_camera(W, H, f, np.eye(3), np.zeros(3))]
        parts = _pack(mean, log_scale, quat, logit, sh, beta, 0)
    elif cfg == 2:
        P = P or 300000
        u = rng.standard_normal((3, P))
        u /= np.linalg.norm(u, axis=0, keepdims=True)
        mean = u * (1.0 + rng.normal(0.0, 0.05, size=P))
        log_scale = rng.normal(-4.5, 0.4, size=(3, P))
        quat = _quats(rng, P)
        logit = rng.normal(0.0, 1.0, size=P)
        beta = rng.uniform(1.0, 6.0, size=P)
        if beta_value is not None:
            beta = np.full(P, beta_value)
        sh = _sh3(rng, P)
        cams = []
        for k in range(8):
            a = 2.0 * math.pi * k / 8.0
            R, t = look_at((4.0 * math.cos(a), 0.0, 4.0 * math.sin(a)))
            cams.append(_camera(800, 800, 1111.1, R, t))
        parts = _pack(mean, log_scale, quat, logit, sh, beta, 3)
    elif cfg in (3, 4):
        P = P or (1500000 if cfg == 3 else 3000000)
        mean = _blob_and_shell(rng, P)
        log_scale = rng.normal(-4.0, 0.8, size=(3, P))
        quat = _quats(rng, P)
        logit = rng.normal(-0.5, 1.5, size=P)
        beta = rng.uniform(0.5, 8.0, size=P)
        if beta_value is not None:
            beta = np.full(P, beta_value)
        sh = _sh3(rng, P)
        parts = _pack(mean, log_scale, quat, logit, sh, beta, 3)
        if cfg == 3:
            # one camera at (0,0,-6) looking down +z (R = I, t = (0,0,6)); extra views
            # for the data-parallel bench orbit the origin at the same radius.
            cams = []
            for k in range(8):
                a = 2.0 * math.pi * k / 8.0
                if k == 0:
                    R, t = np.eye(3), np.array([0.0, 0.0, 6.0])
                else:
                    R, t = look_at((-6.0 * math.sin(a), 0.0, -6.0 * math.cos(a)))
                cams.append(_camera(1297, 840, 1150.0, R, t))
        else:
            cams = []
            crng = np.random.default_rng(seed * 7 + 1)
            for _ in range(64):
                ct = crng.uniform(0.0, 1.0)
                st = math.sqrt(max(0.0, 1.0 - ct * ct))
                ph = crng.uniform(0.0, 2.0 * math.pi)
                c = 6.0 * np.array([st * math.cos(ph), -ct, st * math.sin(ph)])
                R, t = look_at(c)
                cams.append(_camera(1600, 1064, 1418.7, R, t))
    else:
        raise ValueError(f"unknown config {cfg}")
    if n_views is not None:
        cams = cams[:n_views]
    return Scene(CONFIG_NAMES[cfg], parts, cams, rho=0.1, background=(0.0, 0.0, 0.0), seed=seed)


def upstream_grad(scene_seed: int, view: int, W: int, H: int) -> np.ndarray:
    """dL/dimage ~ N(0,1), [3][H][W] float32, seeded per view."""
    rng = np.random.default_rng(scene_seed * 100 + view)
    return rng.standard_normal((3, H, W)).astype(np.float32)


def random_small_scene(seed: int, P: int = 8, W: int = 32, H: int = 32, sh_degree: int = 1,
                       beta_range=(0.5, 6.0), kappa_max: float = 0.9, depth=(3.0, 5.0),
                       log_scale_mu: float = -1.6) -> Scene:
    """Tiny scene for finite-difference pins: a few particles in front of one
    camera, opacities bounded away from the 0.99 clamp."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(depth[0], depth[1], size=P)
    xy = rng.uniform(-0.35, 0.35, size=(2, P)) * z
    mean = np.concatenate([xy, z[None]], axis=0)
    log_scale = rng.normal(log_scale_mu, 0.3, size=(3, P))
    quat = _quats(rng, P)
    kappa = rng.uniform(0.2, kappa_max, size=P)
    logit = np.log(kappa / (1.0 - kappa))
    beta = rng.uniform(beta_range[0], beta_range[1], size=P)
    K = (sh_degree + 1) ** 2
    sh = rng.normal(0.0, 0.2, size=(3 * K, P))
    sh[0:3] = rng.normal(0.6, 0.2, size=(3, P))
    parts = _pack(mean, log_scale, quat, logit, sh, beta, sh_degree)
    f = 0.9 * W
    cam = _camera(W, H, f, np.eye(3), np.zeros(3))
    return Scene(f"small{seed}", parts, [cam], rho=0.1, seed=seed)
