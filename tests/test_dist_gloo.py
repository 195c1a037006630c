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
