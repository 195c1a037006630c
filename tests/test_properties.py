"""Property tests (SURVEY.md §4 "Property tests"): random tiny scenes drawn by
hypothesis.  CPU: the oracle's invariants (Eq. 3: T + sum w = 1, T in [1e-4, 1],
colour in [0, 1] for colours in [0, 1] and a black background; S5 linear in
dL/dimage; a zero upstream gradient gives zero gradients; a background shifts the
image by T bg exactly; sorting is invariant to relabelling particles with distinct
depths).  GPU: the CUDA path = the oracle on the same random scenes (S1 state, keys,
lists bit-exact; image <= 1e-4; every particle's gradients at the north_star
tolerance or their R19 scale)."""
import math

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import ges_inputs as gi
from oracle import oracle as O

SETTINGS = dict(max_examples=25, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@st.composite
def tiny_scene(draw):
    seed = draw(st.integers(0, 2 ** 31 - 1))
    P = draw(st.integers(1, 40))
    W = draw(st.integers(8, 72))
    H = draw(st.integers(8, 56))
    deg = draw(st.integers(0, 3))
    sc = gi.random_small_scene(seed, P=P, W=W, H=H, sh_degree=deg, kappa_max=0.98,
                               log_scale_mu=draw(st.floats(-3.0, -1.0)))
    rho = draw(st.sampled_from([0.0, 0.1, 0.5]))
    return sc, rho


def _white(parts):
    p = parts.subset(slice(None))
    p.sh[:] = 0.0
    p.sh[0:3] = math.sqrt(math.pi)   # Y00 sh = 0.5 -> rgb = 1
    return p


@settings(**SETTINGS)
@given(tiny_scene())
def test_oracle_compositing_invariants(data):
    sc, rho = data
    cam = sc.cameras[0]
    out = O.render(_white(sc.particles), cam, O.Settings(rho=rho), "f64")
    # one colour c for every particle (rgb = Y00 sh + 0.5 = 1 up to the fp32 rounding of sh),
    # black background: image = c sum w = c (1 - T)
    vis = out["pre"]["status"] == O.VISIBLE
    c = float(out["pre"]["rgb"][0, vis][0]) if vis.any() else 1.0
    assert abs(c - 1.0) < 1e-6
    assert np.abs(out["image"][0] / c + out["final_T"] - 1.0).max() < 1e-12
    assert out["final_T"].min() >= np.float32(1e-4) and out["final_T"].max() <= 1.0
    out2 = O.render(sc.particles, cam, O.Settings(rho=rho), "f64")
    rgb = out2["pre"]["rgb"][:, out2["pre"]["status"] == O.VISIBLE]
    if rgb.size and rgb.max() <= 1.0:
        assert out2["image"].min() >= 0.0 and out2["image"].max() <= 1.0 + 1e-12


@settings(**SETTINGS)
@given(tiny_scene(), st.floats(0.0, 1.0), st.floats(0.0, 1.0), st.floats(0.0, 1.0))
def test_oracle_background_adds_T_bg(data, r, g, b):
    sc, rho = data
    cam = sc.cameras[0]
    bg = (r, g, b)
    a = O.render(sc.particles, cam, O.Settings(rho=rho), "f64")
    c = O.render(sc.particles, cam, O.Settings(rho=rho, background=bg), "f64")
    bgc = np.array([np.float32(x) for x in bg], np.float64)[:, None, None]
    assert np.abs(c["image"] - (a["image"] + a["final_T"][None] * bgc)).max() < 1e-12


@settings(**SETTINGS)
@given(tiny_scene(), st.floats(-3.0, 3.0))
def test_oracle_backward_is_linear_in_upstream(data, s):
    sc, rho = data
    cam = sc.cameras[0]
    g = gi.upstream_grad(7, 0, cam.width, cam.height).astype(np.float64)
    a = O.render_and_grad(sc.particles, cam, O.Settings(rho=rho), g)["grads"]
    b = O.render_and_grad(sc.particles, cam, O.Settings(rho=rho), s * g)["grads"]
    for n in a:
        assert np.allclose(b[n], s * a[n], rtol=1e-11, atol=1e-13 * (1 + np.abs(a[n]).max())), n
    z = O.render_and_grad(sc.particles, cam, O.Settings(rho=rho), 0 * g)["grads"]
    assert all(np.all(v == 0.0) for v in z.values())


@settings(**SETTINGS)
@given(tiny_scene(), st.randoms(use_true_random=False))
def test_oracle_relabelling_invariance(data, rnd):
    """Relabelling the particles permutes the lists but changes no pixel (distinct
    depths: the (depth, index) order is the depth order)."""
    sc, rho = data
    cam = sc.cameras[0]
    P = sc.particles.P
    perm = np.arange(P)
    rnd.shuffle(perm)
    a = O.render(sc.particles, cam, O.Settings(rho=rho), "f32")
    depth = a["pre"]["depth"]
    if np.unique(depth.view(np.uint32)).size != P:
        return
    b = O.render(sc.particles.subset(perm), cam, O.Settings(rho=rho), "f32")
    assert np.abs(a["image"] - b["image"]).max() < 1e-12


@pytest.mark.gpu
@settings(max_examples=30, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(tiny_scene(), st.sampled_from([0, 1]))
def test_gpu_equals_oracle_on_random_tiny_scenes(data, kernel):
    import test_parity_gpu as T
    from gpu_helpers import settings_pair
    sc, rho = data
    cam = sc.cameras[0]
    gs, osx = settings_pair(rho=rho, kernel=kernel, background=(0.1, 0.2, 0.3))
    T.run_case(sc.particles, cam, gs, osx, gi.upstream_grad(sc.seed, 0, cam.width, cam.height),
               max_amb_frac=0.05, label=f"random tiny P={sc.particles.P} {cam.width}x{cam.height} kernel={kernel}")
