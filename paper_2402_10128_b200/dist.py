"""Multi-GPU plumbing for view data parallelism.

Particles are replicated on every rank; rank r renders the views assigned to
it (fwd + bwd, gradients accumulated into one flat planar buffer with
`accumulate=1`), then ONE allreduce (sum) over the process group -- NCCL over
NVLink on the B200 box, gloo in the CPU tests.  The gradient of the summed
loss over all views is then identical on every rank.
"""
from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist

from .api import PlanarParams, Renderer, Settings


def views_for_rank(n_views: int, rank: int, world: int) -> List[int]:
    """Round-robin view assignment: rank r gets views r, r + world, ..."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return list(range(rank, n_views, world))


def allreduce_grads(flat: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the flat [C][P] gradient buffer over the group in place (one call)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


class ViewDataParallel:
    """Renders this rank's views of one particle set and returns the
    allreduced parameter gradients of sum_v <dL/dimage_v, image_v>."""

    def __init__(self, params: PlanarParams, cameras: Sequence, settings: Settings, rank: int, world: int,
                 device="cuda", group=None):
        self.params, self.cameras, self.settings = params, list(cameras), settings
        self.views = views_for_rank(len(self.cameras), rank, world)
        self.group = group
        cam0 = self.cameras[0]
        self.renderers = {}
        for v in self.views:
            c = self.cameras[v]
            key = (c.width, c.height)
            if key not in self.renderers:
                self.renderers[key] = Renderer(params.P, c.width, c.height, device=device)
        self.grads = PlanarParams.zeros(params.P, params.sh_degree, device)
        self.images = {}

    def step(self, dL_dimages: dict, stream=None) -> PlanarParams:
        """dL_dimages: view -> [3][H][W] device tensor, for this rank's views."""
        first = True
        for v in self.views:
            cam = self.cameras[v]
            r = self.renderers[(cam.width, cam.height)]
            self.images[v] = r.forward(self.params, cam, self.settings, stream=stream)
            r.backward(self.params, cam, self.settings, dL_dimages[v], grads=self.grads,
                       accumulate=not first, stream=stream)
            first = False
        if first:  # no views on this rank: contribute zeros
            self.grads.flat.zero_()
        allreduce_grads(self.grads.flat, self.group)
        return self.grads
