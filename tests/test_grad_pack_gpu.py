"""GPU checks of the visible-union compaction of the view-DP allreduce (SURVEY.md
§8(e); ges_mask_visible / ges_grad_pack / ges_grad_unpack).  On one GPU two
"ranks" are two views rendered in turn: the mask is the OR of their S1 visible
sets (checked against the oracle's S1 status), the index list is exactly
numpy.nonzero of it, the packed rows are the gradients' columns, and packing
both views' gradients, adding the packed buffers (the allreduce of two ranks)
and unpacking gives bit for bit the dense sum.  The compacted ViewDataParallel
step equals the dense one."""
import numpy as np
import pytest
import torch

import ges_inputs as gi
import paper_2402_10128_b200 as G
from oracle import oracle as O
from paper_2402_10128_b200 import dist as gdist

pytestmark = pytest.mark.gpu


def _zoomed(cam, z=3.0):
    return gi.Camera(cam.width, cam.height, z * cam.fx, z * cam.fy, cam.cx, cam.cy, cam.near, cam.R, cam.t)


def test_pack_unpack_two_views():
    sc = gi.make_config(2, P=20000)
    cams = [_zoomed(sc.cameras[0]), _zoomed(sc.cameras[3])]
    params = G.PlanarParams.from_inputs(sc.particles)
    st = G.Settings(rho=sc.rho)
    red = gdist.VisibleUnionReducer(params.P, params.flat.shape[0])
    grads = []
    for k, cam in enumerate(cams):
        r = G.Renderer(params.P, cam.width, cam.height)
        r.forward(params, cam, st)
        red.add_view(r.frame)
        g = G.PlanarParams.zeros(params.P, params.sh_degree)
        dL = torch.from_numpy(gi.upstream_grad(sc.seed, k, cam.width, cam.height)).cuda()
        r.backward(params, cam, st, dL, grads=g)
        grads.append(g.flat.clone())
    torch.cuda.synchronize()
    vis = [O.preprocess(sc.particles, c, O.Settings(rho=sc.rho), "f32")["status"] == O.VISIBLE for c in cams]
    union = (vis[0] | vis[1]).astype(np.uint8)
    assert np.array_equal(red.mask.cpu().numpy(), union)
    assert 0 < union.sum() < params.P
    packs = []
    for g in grads:
        packed, u = red.pack(g, red.mask, force=True)
        assert u == int(union.sum())
        assert np.array_equal(red.idx[:u].cpu().numpy(), np.nonzero(union)[0])
        cols = g.cpu().numpy()[:, np.nonzero(union)[0]]
        assert np.array_equal(packed.cpu().numpy().reshape(g.shape[0], u), cols)
        packs.append(packed.clone())
    total = packs[0] + packs[1]          # what the allreduce of two ranks computes
    out = torch.zeros_like(grads[0])
    red.unpack(total, None, out)
    torch.cuda.synchronize()
    dense = (grads[0] + grads[1]).cpu().numpy()
    assert np.all(dense[:, union == 0] == 0.0)
    assert np.array_equal(out.cpu().numpy(), dense)


def test_view_data_parallel_compact_equals_dense_single_rank():
    sc = gi.make_config(2, P=20000, n_views=3)
    cams = [_zoomed(c) for c in sc.cameras]
    params = G.PlanarParams.from_inputs(sc.particles)
    st = G.Settings(rho=sc.rho)
    dLs = {v: torch.from_numpy(gi.upstream_grad(sc.seed, v, c.width, c.height)).cuda() for v, c in enumerate(cams)}
    dense = gdist.ViewDataParallel(params, cams, st, 0, 1).step(dLs).flat.clone()
    vdp = gdist.ViewDataParallel(params, cams, st, 0, 1, compact=True)
    vdp.reducer.max_union = 1.0      # always compact (the union here is ~half the particles anyway)
    comp = vdp.step(dLs).flat.clone()
    torch.cuda.synchronize()
    a, b = dense.cpu().numpy(), comp.cpu().numpy()
    # the same accumulation order on one rank; compaction only moves values: equal up to
    # the float atomics of S5a reordering between the two runs
    floor = 1e-6 + 1e-6 * np.abs(a).max()
    assert np.all(np.abs(a - b) <= np.maximum(1e-4 * np.abs(a), floor))


def test_view_data_parallel_sh_factorized_equals_dense_single_rank():
    """ViewDataParallel(sh_factorized=True): the SH planes rebuilt from the views' dL/drgb
    (ges_sh_grad_from_colour) and the untouched non-SH planes equal the dense step's
    gradient; two steps in a row (the drgb slots are re-zeroed)."""
    sc = gi.make_config(2, P=20000, n_views=3)
    cams = [_zoomed(c) for c in sc.cameras]
    params = G.PlanarParams.from_inputs(sc.particles)
    st = G.Settings(rho=sc.rho)
    dLs = {v: torch.from_numpy(gi.upstream_grad(sc.seed, v, c.width, c.height)).cuda() for v, c in enumerate(cams)}
    dense = gdist.ViewDataParallel(params, cams, st, 0, 1).step(dLs).flat.clone()
    vdp = gdist.ViewDataParallel(params, cams, st, 0, 1, sh_factorized=True)
    assert vdp.drgb.shape == (3, 3, params.P)
    for _ in range(2):
        fac = vdp.step(dLs).flat.clone()
        torch.cuda.synchronize()
        a, b = dense.cpu().numpy(), fac.cpu().numpy()
        floor = 1e-6 + 1e-6 * np.abs(a).max()
        assert np.all(np.abs(a - b) <= np.maximum(1e-4 * np.abs(a), floor))
    with pytest.raises(ValueError):
        gdist.ViewDataParallel(params, cams, st, 0, 1, compact=True, sh_factorized=True)


@pytest.mark.parametrize("sh_factorized", [False, True])
def test_view_data_parallel_two_streams(sh_factorized):
    """ViewDataParallel(streams=2): views alternate between two streams and two frames, the
    S5b accumulations serialised in view order; the gradients and images equal the
    one-stream step (float-atomic order aside); frames that overflow are regrown and the
    step redone (one host read of the per-view counters)."""
    sc = gi.make_config(2, P=40000, n_views=5)
    cams = [_zoomed(c) for c in sc.cameras]
    params = G.PlanarParams.from_inputs(sc.particles)
    st = G.Settings(rho=sc.rho)
    dLs = {v: torch.from_numpy(gi.upstream_grad(sc.seed, v, c.width, c.height)).cuda() for v, c in enumerate(cams)}
    one = gdist.ViewDataParallel(params, cams, st, 0, 1, sh_factorized=sh_factorized)
    a = one.step(dLs).flat.clone()
    imgs = {v: one.images[v].clone() for v in one.views}
    two = gdist.ViewDataParallel(params, cams, st, 0, 1, sh_factorized=sh_factorized, streams=2)
    for rl in two.renderers.values():            # too small: the first step must regrow
        for r in rl:
            r.frame = G.Frame(params.P, r.width, r.height, 1024)
    for _ in range(2):
        b = two.step(dLs).flat.clone()
        torch.cuda.synchronize()
        x, y = a.cpu().numpy(), b.cpu().numpy()
        floor = 1e-6 + 1e-6 * np.abs(x).max()
        assert np.all(np.abs(x - y) <= np.maximum(1e-4 * np.abs(x), floor))
        for v in one.views:
            assert torch.equal(imgs[v], two.images[v])
    assert all(r.frame.c.pair_capacity > 1024 for rl in two.renderers.values() for r in rl)
    with pytest.raises(ValueError):
        gdist.ViewDataParallel(params, cams, st, 0, 1, compact=True, streams=2)
