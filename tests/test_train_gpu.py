"""GPU parity of the optimizer and density control against
oracle/train.py: Adam steps within 1e-5 relative of the fp64 update (+1e-6 of the step size), the position
schedule to 1e-12, resets exact, the view-space statistic within the gradient
tolerance, and densify/prune with the same decisions, order and counts (copies
bit-exact; split children within fp32 rounding of the shared generator's draws)."""
import math

import numpy as np
import pytest
import torch

import ges_inputs as gi
import paper_2402_10128_b200 as G
from oracle import oracle as O
from oracle import train as TR

pytestmark = pytest.mark.gpu


def planar(P, deg, seed):
    K = (deg + 1) ** 2
    rng = np.random.default_rng(seed)
    p = rng.normal(0, 1, (12 + 3 * K, P)).astype(np.float32)
    p[3:6] = rng.normal(-3, 0.5, (3, P))
    p[11 + 3 * K] = rng.uniform(0.5, 4, P)
    return p


def to_params(arr, deg):
    t = torch.from_numpy(np.ascontiguousarray(arr, np.float32)).cuda()
    return G.PlanarParams(t, arr.shape[1], deg)


@pytest.mark.parametrize("deg,P", [(3, 10000), (3, 9999), (0, 1), (1, 4097)])
def test_adam_steps_and_schedule(deg, P):
    """P % 4 == 0 takes the float4 kernel, any other P the scalar one."""
    K = (deg + 1) ** 2
    p = planar(P, deg, 1)
    params = to_params(p, deg)
    opt = G.Adam(params)
    ref_p, ref_m, ref_v = p.astype(np.float64), np.zeros((12 + 3 * K, P)), np.zeros((12 + 3 * K, P))
    rng = np.random.default_rng(2)
    for step in range(1, 4):
        g = rng.normal(0, 1e-3, p.shape).astype(np.float32)
        opt.step(params, to_params(g, deg))
        ref_p, ref_m, ref_v = TR.adam_step(ref_p, g.astype(np.float64), ref_m, ref_v, step, K)
    torch.cuda.synchronize()
    got = params.flat.cpu().numpy().astype(np.float64)
    delta_ref = ref_p - p.astype(np.float64)
    delta_got = got - p.astype(np.float64)
    # fp32 moments: m = beta1 m + (1 - beta1) g cancels when g changes sign, so the bar is
    # 1e-5 of the update plus 1e-6 of the plane's step size, plus fp32 rounding of p
    lr = TR.plane_lrs(K, 3)[:, None]
    assert np.all(np.abs(delta_got - delta_ref) <= 1e-5 * np.abs(delta_ref) + 1e-6 * lr + 4e-7 * np.abs(p))
    s = G.AdamSettings()
    for step in (0, 1, 777, 15000, 30000, 45000):
        assert abs(s.lr_position(step) - TR.lr_position(step)) <= 1e-12 * TR.lr_position(step)


def test_resets_exact():
    deg, P = 1, 5000
    K = (deg + 1) ** 2
    p = planar(P, deg, 3)
    p[10, :100] = 6.0
    params = to_params(p, deg)
    G.ges_reset(params, 0)
    cap = np.float32(math.log(0.01 / 0.99))
    got = params.flat.cpu().numpy()
    assert np.array_equal(got[10], np.minimum(p[10], cap))
    G.ges_reset(params, 1)
    got = params.flat.cpu().numpy()
    assert np.all(got[11 + 3 * K] == 2.0)
    assert np.array_equal(np.delete(got, [10, 11 + 3 * K], axis=0), np.delete(p, [10, 11 + 3 * K], axis=0))


def test_densify_statistic_matches_viewspace_gradient():
    sc = gi.make_config(0, P=1500)
    cam = sc.cameras[0]
    params = G.PlanarParams.from_inputs(sc.particles)
    st = G.Settings(rho=0.1)
    r = G.Renderer(params.P, cam.width, cam.height)
    r.forward(params, cam, st)
    dL = gi.upstream_grad(sc.seed, 0, cam.width, cam.height)
    dc = G.DensityControl(params.P)
    G.ges_render_bwd_tiles(st, r.frame, torch.from_numpy(dL).cuda())
    dc.accumulate(r.frame)
    grads = G.PlanarParams.zeros(params.P, params.sh_degree)
    G.ges_backward_particles(params, cam, st, r.frame, grads)
    torch.cuda.synchronize()
    pre = O.preprocess(sc.particles, cam, O.Settings(rho=0.1), "f32")
    g2d = O.render_bwd(pre, cam, O.Settings(rho=0.1), *O.tile_lists(pre), dL)
    ref = TR.viewspace_grad_norm(g2d[0], g2d[1], cam.width, cam.height)
    vis = pre["status"] == 0
    acc, cnt = dc.accum.cpu().numpy(), dc.count.cpu().numpy()
    assert np.array_equal(cnt, vis.astype(np.float32))
    assert np.all(np.abs(acc - ref) <= 1e-3 * np.abs(ref) + 1e-6 * np.abs(ref).max())


def test_densify_prune_parity():
    deg, P = 1, 3000
    K = (deg + 1) ** 2
    rng = np.random.default_rng(5)
    p = planar(P, deg, 4)
    p[10] = rng.normal(1, 2.5, P)                       # some kappa < 0.005 (logit < -5.3)
    p[11 + 3 * K, :40] = -20.0                          # phi-bar < 0.5 -> pruned
    p[3:6] = rng.normal(math.log(0.05), 0.8, (3, P))    # around the clone/split boundary (0.01 x 10)
    acc = rng.uniform(0, 6e-4, P).astype(np.float32)
    cnt = rng.integers(0, 3, P).astype(np.float32)
    params = to_params(p, deg)
    opt = G.Adam(params)
    m = rng.normal(0, 1e-3, p.shape).astype(np.float32)
    v = np.abs(rng.normal(0, 1e-6, p.shape)).astype(np.float32)
    opt.m.flat.copy_(torch.from_numpy(m))
    opt.v.flat.copy_(torch.from_numpy(v))
    dc = G.DensityControl(P)
    dc.accum.copy_(torch.from_numpy(acc))
    dc.count.copy_(torch.from_numpy(cnt))
    ds = G.DensitySettings(scene_extent=10.0, rho=0.1, seed=11)
    newp = dc.densify_prune(params, opt, ds)
    torch.cuda.synchronize()
    q, mq, vq, act = TR.densify_prune(p.astype(np.float64), m.astype(np.float64), v.astype(np.float64),
                                      acc.astype(np.float64), cnt.astype(np.float64), K, 10.0, 0.1, 11)
    assert (act == 0).sum() > 40 and (act == 2).sum() > 10 and (act == 3).sum() > 10
    assert newp.P == q.shape[1]
    got, gm, gv = newp.flat.cpu().numpy(), opt.m.flat.cpu().numpy(), opt.v.flat.cpu().numpy()
    nk = int((act > 0).sum())
    split_cols = [j for j, i in enumerate(np.nonzero(act > 0)[0]) if act[i] == 3]
    second = list(range(q.shape[1] - int((act == 3).sum()), q.shape[1]))
    exact = np.setdiff1d(np.arange(q.shape[1]), split_cols + second)
    assert np.array_equal(got[:, exact], q[:, exact].astype(np.float32))
    assert np.array_equal(gm[:, exact], mq[:, exact].astype(np.float32))
    assert np.array_equal(gv[:, exact], vq[:, exact].astype(np.float32))
    cols = split_cols + second
    assert np.allclose(got[0:3, cols], q[0:3, cols], rtol=0, atol=2e-5)
    assert np.allclose(got[3:6, cols], q[3:6, cols], rtol=0, atol=2e-6)
    assert np.array_equal(got[6:, cols], q[6:, cols].astype(np.float32))
    assert not gm[:, cols].any() and not gv[:, cols].any()
    assert nk + int((act == 2).sum()) + int((act == 3).sum()) == q.shape[1]


@pytest.mark.parametrize("deg,P,world", [(3, 10000, 8), (3, 9999, 3), (1, 4097, 2)])
def test_adam_step_range_equals_full_step(deg, P, world):
    """ges_adam_step_range (the ZeRO-1 shard update of dist.ShardedAdam) on every rank's
    range of the flat buffer reproduces ges_adam_step bit for bit, ranges straddling
    plane boundaries included (float4 and scalar kernels)."""
    from paper_2402_10128_b200 import dist as gdist
    p = planar(P, deg, 3)
    g = planar(P, deg, 4)
    full, parts = to_params(p, deg), to_params(p, deg)
    grads = to_params(g, deg)
    opt_full, opt_parts = G.Adam(full), G.Adam(parts)
    for step in range(3):
        opt_full.step(full, grads)
        n = parts.flat.numel()
        for r in range(world):
            b, c, _ = gdist.shard_range(n, r, world)
            opt_parts.step_range(parts, grads.flat.view(-1)[b:b + c].contiguous(), b, c)
            opt_parts.t -= 1
        opt_parts.t += 1
    torch.cuda.synchronize()
    assert torch.equal(full.flat, parts.flat)
    assert torch.equal(opt_full.m.flat, opt_parts.m.flat) and torch.equal(opt_full.v.flat, opt_parts.v.flat)
