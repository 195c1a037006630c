"""World-size-2 gloo test of the view-data-parallel host logic (CPU).

Each rank takes its views (dist.views_for_rank), computes the per-view
particle gradients (here with the oracle: the CUDA kernels need a GPU),
accumulates them into one flat planar fp32 buffer and calls the product's
allreduce_grads.  Every rank must end with the gradient of the summed loss
over all views, equal to the single-process sum (linearity).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ges_inputs as gi
from oracle import oracle as O
from paper_2402_10128_b200 import dist as gdist

N_VIEWS = 3


def _scene():
    return gi.make_config(2, P=400, n_views=N_VIEWS)


def _flat(grads, K):
    return np.concatenate([grads["mean"], grads["log_scale"], grads["quat"], grads["opacity_logit"][None],
                           grads["sh"], grads["beta"][None]], axis=0).astype(np.float32)


def _view_grads(sc, v):
    cam = sc.cameras[v]
    cam = gi.Camera(96, 96, cam.fx * 96 / 800, cam.fy * 96 / 800, 48.0, 48.0, cam.near, cam.R, cam.t)
    g = gi.upstream_grad(sc.seed, v, 96, 96)
    r = O.render_and_grad(sc.particles, cam, O.Settings(), g)
    return _flat(r["grads"], sc.particles.K)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = _scene()
        views = gdist.views_for_rank(N_VIEWS, rank, world)
        flat = torch.zeros((sc.particles.n_planes(), sc.particles.P), dtype=torch.float32)
        for v in views:
            flat += torch.from_numpy(_view_grads(sc, v))
        gdist.allreduce_grads(flat)
        out[rank] = flat.numpy().copy()
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_views_for_rank_partition():
    for world in (1, 2, 3, 8):
        got = sorted(v for r in range(world) for v in gdist.views_for_rank(64, r, world))
        assert got == list(range(64))
    with pytest.raises(ValueError):
        gdist.views_for_rank(4, 2, 2)


def test_allreduce_of_view_gradients_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    sc = _scene()
    ref = sum(_view_grads(sc, v).astype(np.float64) for v in range(N_VIEWS))
    for r in range(world):
        assert np.allclose(out[r], ref, rtol=1e-5, atol=1e-6)
    assert np.array_equal(out[0], out[1])


# --------------------------------------------------------------------------
# screen-tile bands: rank r owns tile rows r, r + N, ...
# --------------------------------------------------------------------------
BAND_W, BAND_H = 96, 72   # 5 tile rows: rank 0 -> rows 0, 2, 4; rank 1 -> rows 1, 3


def _band_scene():
    sc = gi.make_config(2, P=400, n_views=1)
    c = sc.cameras[0]
    cam = gi.Camera(BAND_W, BAND_H, c.fx * BAND_W / 800, c.fy * BAND_W / 800, BAND_W / 2, BAND_H / 2, c.near, c.R,
                    c.t)
    return sc, cam


def _band_mask(rank, world):
    ty, tx = (BAND_H + 15) // 16, (BAND_W + 15) // 16
    m = np.zeros((ty, tx), np.uint8)
    m[rank::world] = 1
    return m.reshape(-1)


def _band_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, cam = _band_scene()
        g = gi.upstream_grad(sc.seed, 0, BAND_W, BAND_H)
        r = O.render_and_grad(sc.particles, cam, O.Settings(), g, tile_mask=_band_mask(rank, world))
        img = torch.full((3, BAND_H, BAND_W), float("nan"), dtype=torch.float64)
        rows = gdist.band_pixel_rows(BAND_H, rank, world)
        img[:, rows] = torch.from_numpy(np.ascontiguousarray(r["image"]))[:, rows]
        full = gdist.gather_bands(img, rank, world)
        flat = torch.from_numpy(_flat(r["grads"], sc.particles.K))
        gdist.allreduce_grads(flat)
        out[rank] = (full.numpy().copy(), flat.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_band_rows_partition_the_image():
    for H in (16, 72, 840, 1000):
        for world in (1, 2, 3, 8):
            got = torch.cat([gdist.band_pixel_rows(H, r, world) for r in range(world)]).sort().values
            assert torch.equal(got, torch.arange(H))
    assert gdist.band_settings(gdist.Settings(), 1, 4).tile_row_begin == 1


def test_band_gather_and_gradient_allreduce_world2():
    """The gathered band image is the full-frame image exactly; the allreduced
    per-band gradients sum to the full-frame gradient (linearity of S5)."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_band_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    sc, cam = _band_scene()
    g = gi.upstream_grad(sc.seed, 0, BAND_W, BAND_H)
    ref = O.render_and_grad(sc.particles, cam, O.Settings(), g)
    ref_flat = _flat(ref["grads"], sc.particles.K).astype(np.float64)
    assert np.abs(ref_flat).max() > 0
    for r in range(world):
        img, flat = out[r]
        assert np.array_equal(img, ref["image"])
        assert np.allclose(flat, ref_flat, rtol=1e-5, atol=1e-6)


# --------------------------------------------------------------------------
# visible-union compaction of the view-DP allreduce
# --------------------------------------------------------------------------
def _view_grads_and_mask(sc, v):
    cam = sc.cameras[v]   # zoomed in 3x: each view sees part of the object
    cam = gi.Camera(96, 96, 3 * cam.fx * 96 / 800, 3 * cam.fy * 96 / 800, 48.0, 48.0, cam.near, cam.R, cam.t)
    g = gi.upstream_grad(sc.seed, v, 96, 96)
    r = O.render_and_grad(sc.particles, cam, O.Settings(), g)
    pre = O.preprocess(sc.particles, cam, O.Settings(), "f32")
    return _flat(r["grads"], sc.particles.K), (pre["status"] == O.VISIBLE).astype(np.uint8)


def _np_pack(flat, mask):
    idx = np.nonzero(mask.numpy())[0]
    return torch.from_numpy(np.ascontiguousarray(flat.numpy()[:, idx]).reshape(-1)), idx


def _np_unpack(packed, idx, flat):
    flat.numpy()[:, idx] = packed.numpy().reshape(flat.shape[0], idx.size)


def _union_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = _scene()
        flat = torch.zeros((sc.particles.n_planes(), sc.particles.P), dtype=torch.float32)
        mask = torch.zeros(sc.particles.P, dtype=torch.uint8)
        for v in gdist.views_for_rank(N_VIEWS, rank, world):
            g, m = _view_grads_and_mask(sc, v)
            flat += torch.from_numpy(g)
            mask |= torch.from_numpy(m)
        local_mask = mask.clone()
        gdist.allreduce_visible_union(flat, mask, _np_pack, _np_unpack)
        out[rank] = (flat.numpy().copy(), mask.numpy().copy(), local_mask.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_visible_union_allreduce_world2():
    """The compacted allreduce equals the dense one: every rank ends with the sum over
    all views, the union mask is the OR of the ranks' masks, and no gradient outside
    the union is nonzero anywhere (what makes the compaction exact)."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_union_worker, args=(world, port, out), nprocs=world, join=True)
    sc = _scene()
    gs = [_view_grads_and_mask(sc, v) for v in range(N_VIEWS)]
    ref = sum(g.astype(np.float64) for g, _ in gs)
    union = np.zeros(sc.particles.P, np.uint8)
    for _, m in gs:
        union |= m
    assert np.all(ref[:, union == 0] == 0.0)
    assert 0 < union.sum() < sc.particles.P
    for r in range(world):
        flat, mask, local = out[r]
        assert np.array_equal(mask, union)
        assert np.allclose(flat, ref, rtol=1e-5, atol=1e-6)
    assert np.array_equal(out[0][0], out[1][0])
    assert not np.array_equal(out[0][2], out[1][2])   # the ranks saw different particles


# --------------------------------------------------------------------------
# DP-consistent density control
# --------------------------------------------------------------------------
from oracle import train as TR  # noqa: E402

DENS_VIEWS = 4


def _density_scene():
    sc = gi.make_config(2, P=600, n_views=DENS_VIEWS)
    K = sc.particles.K
    params = np.concatenate([sc.particles.mean, sc.particles.log_scale, sc.particles.quat,
                             sc.particles.opacity_logit[None], sc.particles.sh, sc.particles.beta[None]],
                            axis=0).astype(np.float64)
    # a few particles large and dense enough to split, a few faint enough to prune
    params[3:6, :40] += 3.0
    params[10, 40:60] = -8.0
    return sc, params, K


def _view_stats(sc, v):
    """One view's contribution to the densification statistic (R32): the view-space
    gradient norm |(du W/2, dv H/2)| of every particle the view saw, and a count of 1."""
    cam = sc.cameras[v]
    cam = gi.Camera(96, 96, 2 * cam.fx * 96 / 800, 2 * cam.fy * 96 / 800, 48.0, 48.0, cam.near, cam.R, cam.t)
    g = gi.upstream_grad(sc.seed, v, 96, 96)
    r = O.render_and_grad(sc.particles, cam, O.Settings(), g)
    vis = r["pre"]["status"] == O.VISIBLE
    norm = TR.viewspace_grad_norm(r["g2d"][0], r["g2d"][1], 96, 96)
    return np.where(vis, norm, 0.0).astype(np.float32), vis.astype(np.float32)


def _density_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, params, K = _density_scene()
        accum = torch.zeros(sc.particles.P, dtype=torch.float32)
        count = torch.zeros(sc.particles.P, dtype=torch.float32)
        for v in gdist.views_for_rank(DENS_VIEWS, rank, world):
            a, c = _view_stats(sc, v)
            accum += torch.from_numpy(a)
            count += torch.from_numpy(c)
        local = TR.densify_prune(params, np.zeros_like(params), np.zeros_like(params), accum.numpy().astype(np.float64),
                                 count.numpy().astype(np.float64), K, 1.0, 0.1, 7)[0]
        gdist.allreduce_density_stats(accum, count)
        new = TR.densify_prune(params, np.zeros_like(params), np.zeros_like(params), accum.numpy().astype(np.float64),
                               count.numpy().astype(np.float64), K, 1.0, 0.1, 7)
        out[rank] = (new[0], new[3], local, accum.numpy().copy(), count.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_density_control_is_identical_on_every_rank_world2():
    """Clone / split / prune decisions come from the view-space gradient statistics
    summed over ALL ranks' views (dist.allreduce_density_stats): both ranks produce
    bit-identical densified sets, equal to a single process that saw every view --
    while densifying on the local statistics alone would make the ranks diverge."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_density_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    sc, params, K = _density_scene()
    stats = [_view_stats(sc, v) for v in range(DENS_VIEWS)]
    accum = sum(a.astype(np.float64) for a, _ in stats)
    count = sum(c.astype(np.float64) for _, c in stats)
    ref = TR.densify_prune(params, np.zeros_like(params), np.zeros_like(params), accum, count, K, 1.0, 0.1, 7)
    acts = ref[3]
    assert (acts == 0).any() and (acts == 3).any() and (acts == 1).any()   # prune, split, keep all occur
    for r in range(world):
        new, act, _, a, c = out[r]
        assert np.allclose(a, accum, rtol=1e-6, atol=1e-9) and np.array_equal(c, count)
        assert np.array_equal(act, acts)
        assert np.array_equal(new, ref[0])
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][2].shape != out[1][2].shape or not np.array_equal(out[0][2], out[1][2])  # local stats diverge


# --------------------------------------------------------------------------
# ZeRO-1 sharded optimizer step of the view-DP training step (dist.sharded_update)
# --------------------------------------------------------------------------
def _zero1_problem(sh_degree, P):
    K = (sh_degree + 1) ** 2
    C = 12 + 3 * K
    rng = np.random.default_rng(11)
    params = rng.normal(0, 1, (C, P))
    local = [rng.normal(0, 1, (C, P)) for _ in range(2)]   # each rank's accumulated view gradients
    return K, C, params, local


def _zero1_worker(rank, world, port, sh_degree, P, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, C, params0, local = _zero1_problem(sh_degree, P)
        params = torch.from_numpy(params0.copy())
        state = {"m": np.zeros((C, P)), "v": np.zeros((C, P)), "t": 0}

        def update(gshard, begin, count):
            # the oracle Adam (elementwise) on the flat range only
            state["t"] += 1
            g = np.zeros(C * P)
            g[begin:begin + count] = gshard.numpy()[:count]
            p2, m2, v2 = TR.adam_step(params.numpy().reshape(C, P), g.reshape(C, P), state["m"], state["v"],
                                      state["t"], K)
            sl = slice(begin, begin + count)
            params.view(-1)[sl] = torch.from_numpy(p2.reshape(-1)[sl])
            state["m"].reshape(-1)[sl] = m2.reshape(-1)[sl]
            state["v"].reshape(-1)[sl] = v2.reshape(-1)[sl]

        scratch = {}
        for s in range(steps):
            grads = torch.from_numpy(local[rank] * (1.0 + 0.1 * s))
            gdist.sharded_update(grads.reshape(-1), params.view(-1), update, rank, world, scratch=scratch)
        out[rank] = params.numpy().copy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sh_degree,P", [(3, 40), (0, 37)])   # C P even / odd (padded collectives)
def test_zero1_sharded_update_world2(sh_degree, P):
    """Reduce-scatter + per-shard Adam + all-gather (ZeRO-1) gives every rank the
    parameters of a single process running Adam on the summed gradients."""
    world, steps = 2, 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_zero1_worker, args=(world, _free_port(), sh_degree, P, steps, out), nprocs=world, join=True)
    K, C, params, local = _zero1_problem(sh_degree, P)
    m, v = np.zeros((C, P)), np.zeros((C, P))
    for s in range(steps):
        g = (local[0] + local[1]) * (1.0 + 0.1 * s)
        params, m, v = TR.adam_step(params, g, m, v, s + 1, K)
    for r in range(world):
        assert np.allclose(out[r], params, rtol=1e-12, atol=1e-12)
    assert np.array_equal(out[0], out[1])
    begin0, c0, shard = gdist.shard_range(C * P, 0, world)
    begin1, c1, _ = gdist.shard_range(C * P, 1, world)
    assert begin0 == 0 and begin1 == shard and c0 + c1 == C * P


# --------------------------------------------------------------------------
# SH-factorised exchange: all-gather the per-view dL/drgb, reduce
# the 12 non-SH planes, rebuild the SH planes locally
# --------------------------------------------------------------------------
SHF_DEG, SHF_P, SHF_V = 2, 37, 3   # 3 views per rank


def _fake_sh_from_colour(d_all, c_all, out):
    """A stand-in for ges_sh_grad_from_colour with the same linear structure:
    out[3k + ch] = sum_v basis(c_v)[k] drgb_v[ch] (basis: a fixed function of the view's camera row)."""
    K = out.shape[0] // 3
    out.zero_()
    for v in range(d_all.shape[0]):
        basis = torch.cos(c_all[v, :K] * 3.0 + torch.arange(K, dtype=torch.float32))
        for k in range(K):
            out[3 * k:3 * k + 3] += basis[k] * d_all[v]


def _shf_rank_data(rank):
    g = torch.Generator().manual_seed(100 + rank)
    C = 3 + 3 + 4 + 1 + 3 * (SHF_DEG + 1) ** 2 + 1
    flat = torch.randn((C, SHF_P), generator=g)
    drgb = torch.randn((SHF_V, 3, SHF_P), generator=g)
    drgb[:, :, ::5] = 0.0                       # particles a view did not see
    cams = torch.randn((SHF_V, 12), generator=g)
    lo, hi = gdist.sh_rows(SHF_DEG)
    _fake_sh_from_colour(drgb, cams, flat[lo:hi])   # the rank's own SH planes (what S5b accumulates)
    return flat, drgb, cams


def _shf_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        flat, drgb, cams = _shf_rank_data(rank)
        dense = flat.clone()
        dist.all_reduce(dense)
        gdist.allreduce_grads_sh_factorized(flat, SHF_DEG, drgb, cams,
                                            lambda d, c, o: _fake_sh_from_colour(d, c, o))
        out[rank] = (flat.numpy().copy(), dense.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_sh_factorized_exchange_world2():
    """The factorised exchange gives every rank the dense allreduce's sum: non-SH planes
    reduced, SH planes rebuilt from the gathered per-view colour gradients (sum order
    differs: fp32 tolerance), bit-identical across the ranks."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shf_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        got, dense = out[r]
        assert np.allclose(got, dense, rtol=1e-5, atol=1e-5)
    assert np.array_equal(out[0][0], out[1][0])
    lo, hi = gdist.sh_rows(SHF_DEG)
    assert (lo, hi) == (11, 11 + 27)
