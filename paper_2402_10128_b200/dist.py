"""Multi-GPU plumbing.

View data parallelism: particles are replicated on every rank; rank r renders
the views assigned to it (fwd + bwd, gradients accumulated into one flat planar
buffer with `accumulate=1`), then ONE allreduce (sum) over the process group --
NCCL over NVLink on the B200 box, gloo in the CPU tests.  The gradient of the
summed loss over all views is then identical on every rank.

Screen-tile bands (BASELINE config 3: "the 8 GPUs splitting screen-tile bands
of one frame"): rank r renders the tile rows r, r + N, r + 2N, ... of the same
frame (interleaved for load balance; ges_settings tile_row_begin/step), then
the band pixels are all-gathered into the full image.  The per-tile lists and
pixels of a band are the full frame's, so the gathered image is bit-identical
to a one-GPU render; for fwd+bwd the per-band particle gradients are summed
with the same allreduce.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

from . import _lib as L
from .api import (Frame, PlanarParams, Renderer, Settings, _stream, ges_backward_particles,
                  ges_render_bwd_tiles, sh_grad_from_colour)

TILE = 16


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


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


def sh_rows(sh_degree: int):
    """Rows of the planar [C][P] buffer holding the SH planes (mean 3, log-scale 3, quat 4,
    logit 1, then the 3K SH planes, then beta)."""
    K = (sh_degree + 1) ** 2
    return 11, 11 + 3 * K


def allreduce_grads_sh_factorized(flat: torch.Tensor, sh_degree: int, drgb: torch.Tensor, cams: torch.Tensor,
                                  sh_from_colour, group=None) -> torch.Tensor:
    """View-DP gradient exchange with the SH gradient factorised.  The SH
    gradient of a view is Y_k(u_v) dL/drgb_v per particle (S5b's own expression), so
    instead of reducing the 3K SH planes each rank all-gathers the 3-float dL/drgb of its
    views (drgb [V][3][P], ges_grads.drgb) and their cameras (cams [V][12]), reduces only
    the 12 non-SH planes, and rebuilds the SH planes of the summed gradient locally with
    sh_from_colour(drgb_all [n][3][P], cams_all [n][12], out_sh [3K][P]) (the GPU path:
    ges_sh_grad_from_colour; the same call on every rank, so the result is identical on
    all of them).  Bytes per particle received per rank: 4 (12 + 3 V (N - 1)) instead of
    the 4 (12 + 3K) of the full buffer's reduction (N ranks, V views each)."""
    lo, hi = sh_rows(sh_degree)
    C = flat.shape[0]
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rest = torch.cat([flat[:lo], flat[hi:]]) if world > 1 else None
    if world > 1:
        dist.all_reduce(rest, op=dist.ReduceOp.SUM, group=group)
        flat[:lo].copy_(rest[:lo])
        flat[hi:].copy_(rest[lo:])
        d_all = torch.empty((world * drgb.shape[0],) + tuple(drgb.shape[1:]), dtype=drgb.dtype, device=drgb.device)
        c_all = torch.empty((world * cams.shape[0], cams.shape[1]), dtype=cams.dtype, device=cams.device)
        dist.all_gather_into_tensor(d_all, drgb.contiguous(), group=group)
        dist.all_gather_into_tensor(c_all, cams.contiguous(), group=group)
    else:
        d_all, c_all = drgb, cams
    sh_from_colour(d_all.contiguous(), c_all.contiguous(), flat[lo:hi])
    assert flat.shape[0] == C
    return flat


def allreduce_density_stats(accum: torch.Tensor, count: torch.Tensor, group=None) -> None:
    """Sum the densification statistics (DensityControl.accum / .count: the per-particle
    view-space gradient norms and the number of views that saw each particle) over the
    group in place, so that every data-parallel rank takes the same clone / split /
    prune decisions.  The mean over the
    views a particle was visible in, accum / count, is then the global one: with the
    parameters and Adam moments already identical on every rank (the gradients are
    allreduced) and the split draws counter-based (seeded, R32), the
    densified sets are bit-identical."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        both = torch.stack([accum, count])
        dist.all_reduce(both, op=dist.ReduceOp.SUM, group=group)
        accum.copy_(both[0])
        count.copy_(both[1])


def allreduce_visible_union(flat: torch.Tensor, mask: torch.Tensor, pack, unpack, group=None) -> torch.Tensor:
    """Visible-union compaction of the view-DP allreduce: OR the
    ranks' visibility masks (a MAX allreduce of P bytes), pack the gradient rows of
    the union, allreduce only those C U floats, unpack.  Particles outside the union
    have zero gradient on every rank, so the result equals the dense allreduce.
    pack(flat, mask) -> (packed 1-D tensor of C U floats, or None when the union is
    too large for compaction to pay -- then the dense buffer is reduced -- , state);
    unpack(packed, state, flat) writes the reduced rows back."""
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    if world > 1:
        dist.all_reduce(mask, op=dist.ReduceOp.MAX, group=group)
    packed, state = pack(flat, mask)
    if packed is None:
        return allreduce_grads(flat, group)
    if world > 1 and packed.numel():
        dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    unpack(packed, state, flat)
    return flat


class VisibleUnionReducer:
    """Device buffers and the CUDA pack / unpack (ges_mask_visible, ges_grad_pack,
    ges_grad_unpack) for allreduce_visible_union over a planar [C][P] gradient."""

    def __init__(self, P: int, n_planes: int, device="cuda", max_union: float = 0.5):
        # compaction moves 4 C U bytes twice on each rank to save 4 C (P - U) on the wire:
        # above max_union P the dense allreduce is used
        self.P, self.C, self.max_union = P, n_planes, max_union
        self.mask = torch.zeros(P, dtype=torch.uint8, device=device)
        self.idx = torch.empty(P, dtype=torch.int32, device=device)
        self.U = torch.zeros(1, dtype=torch.int64, device=device)
        self.packed = torch.empty(n_planes * P, dtype=torch.float32, device=device)
        self.ws = torch.empty(max(1, L.load().ges_grad_pack_workspace_bytes(P)), dtype=torch.uint8, device=device)

    def reset(self) -> None:
        self.mask.zero_()

    def add_view(self, frame: Frame, stream=None) -> None:
        """Marks the particles the frame's last ges_preprocess found visible."""
        L.check(L.load().ges_mask_visible(C.byref(frame.c), C.c_void_p(self.mask.data_ptr()),
                                          C.c_void_p(_stream(stream))), "ges_mask_visible")

    def index(self, mask: torch.Tensor, stream=None) -> None:
        """Device-only: idx = the union's particles in order, U = their count (no host read)."""
        L.check(L.load().ges_grad_index(self.P, C.c_void_p(mask.data_ptr()), C.c_void_p(self.ws.data_ptr()),
                                        self.ws.numel(), C.c_void_p(self.idx.data_ptr()),
                                        C.c_void_p(self.U.data_ptr()), C.c_void_p(_stream(stream))),
                "ges_grad_index")

    def pack_indexed(self, flat: torch.Tensor, stream=None) -> torch.Tensor:
        """Device-only: the C U gradient floats of the indexed union into self.packed."""
        L.check(L.load().ges_grad_pack(C.c_void_p(flat.data_ptr()), self.P, self.C, C.c_void_p(self.idx.data_ptr()),
                                       C.c_void_p(self.U.data_ptr()), C.c_void_p(self.packed.data_ptr()),
                                       C.c_void_p(_stream(stream))), "ges_grad_pack")
        return self.packed

    def pack(self, flat: torch.Tensor, mask: torch.Tensor, stream=None, force: bool = False):
        """Index, then ONE host read of U (it decides dense vs compact and sizes the
        collective -- so a compact step is not graph-capturable, and on view sets that
        cover most particles, e.g. the 8 config-3 bench views at 79 %, the dense
        allreduce is cheaper: compact=True pays off for sparse-coverage view sets)."""
        self.index(mask, stream)
        u = int(self.U.item())
        if not force and u > self.max_union * self.P:
            return None, u
        self.pack_indexed(flat, stream)
        return self.packed[: self.C * u], u

    def unpack(self, packed: torch.Tensor, state, flat: torch.Tensor, stream=None) -> None:
        L.check(L.load().ges_grad_unpack(C.c_void_p(packed.data_ptr()), self.P, self.C,
                                         C.c_void_p(self.idx.data_ptr()), C.c_void_p(self.U.data_ptr()),
                                         C.c_void_p(flat.data_ptr()), C.c_void_p(_stream(stream))),
                "ges_grad_unpack")

    def allreduce(self, flat: torch.Tensor, group=None) -> torch.Tensor:
        return allreduce_visible_union(flat, self.mask, self.pack, self.unpack, group)


def shard_range(n: int, rank: int, world: int):
    """ZeRO-1 shard of a flat buffer of n elements: (begin, count, shard) with shard =
    ceil(n / world) (the padded per-rank size of the collectives)."""
    shard = -(-n // world)
    begin = min(n, rank * shard)
    return begin, max(0, min(shard, n - begin)), shard


def sharded_update(grads_flat: torch.Tensor, params_flat: torch.Tensor, update, rank: int, world: int,
                   group=None, scratch: Optional[dict] = None) -> None:
    """The data-parallel optimizer step with the optimizer sharded over the ranks
    (ZeRO-1): reduce-scatter the gradient buffer (rank r receives the SUM over ranks of
    its 1/N range), update only that range (`update(grad_range, begin, count)`), then
    all-gather the updated ranges so every rank holds the full new parameters.  The
    same bytes cross NVLink as with one allreduce, but the O(P) optimizer work (Adam
    reads and writes 28 B per element) is split N ways instead of replicated.
    grads_flat / params_flat: the flat [C P] views (contiguous)."""
    n = params_flat.numel()
    begin, count, shard = shard_range(n, rank, world)
    scratch = scratch if scratch is not None else {}
    if world == 1:
        update(grads_flat, 0, n)
        return
    padded = shard * world != n
    if padded:  # the collectives need world equal pieces
        if "g" not in scratch:
            scratch["g"] = torch.zeros(shard * world, dtype=grads_flat.dtype, device=grads_flat.device)
            scratch["p"] = torch.zeros(shard * world, dtype=params_flat.dtype, device=params_flat.device)
        gsrc, pbuf = scratch["g"], scratch["p"]
        gsrc[:n].copy_(grads_flat)
    else:
        gsrc, pbuf = grads_flat, params_flat
    if "gs" not in scratch:
        scratch["gs"] = torch.empty(shard, dtype=grads_flat.dtype, device=grads_flat.device)
    gshard = scratch["gs"]
    dist.reduce_scatter_tensor(gshard, gsrc, op=dist.ReduceOp.SUM, group=group)
    update(gshard, begin, count)
    if padded:
        pbuf[begin:begin + count].copy_(params_flat[begin:begin + count])
    # in place: this rank's input is its own range of the output
    dist.all_gather_into_tensor(pbuf, pbuf[rank * shard:(rank + 1) * shard], group=group)
    if padded:
        params_flat.copy_(pbuf[:n])


class ShardedAdam:
    """Adam for view-data-parallel training with ZeRO-1 optimizer sharding
    (sharded_update): every rank keeps the full moments (simple; the saving is the
    update work, 28 B per parameter element, done once per element across the ranks
    instead of on every rank) and updates its 1/N range of the flat parameters."""

    def __init__(self, params: PlanarParams, settings=None, rank: int = 0, world: int = 1, group=None):
        from .api import Adam
        self.adam = Adam(params, settings)
        self.rank, self.world, self.group = rank, world, group
        self.scratch = {}

    def step(self, params: PlanarParams, grads: PlanarParams, stream=None) -> None:
        """Call on torch's current stream (the collectives run there)."""
        if self.world == 1:
            self.adam.step(params, grads, stream)
            return
        sharded_update(grads.flat.view(-1), params.flat.view(-1),
                       lambda g, b, c: self.adam.step_range(params, g, b, c, stream), self.rank, self.world,
                       self.group, self.scratch)


class ViewDataParallel:
    """Renders this rank's views of one particle set and returns the
    allreduced parameter gradients of sum_v <dL/dimage_v, image_v>."""

    def __init__(self, params: PlanarParams, cameras: Sequence, settings: Settings, rank: int, world: int,
                 device="cuda", group=None, compact: bool = False, sh_factorized: bool = False, streams: int = 1):
        self.params, self.cameras, self.settings = params, list(cameras), settings
        if compact and sh_factorized:
            raise ValueError("compact and sh_factorized are alternative exchanges")
        # streams = 2: consecutive views alternate between two streams and two frames, so one
        # view's latency-bound phases (sort, render tails) overlap the other's; the S5b
        # accumulations into the one gradient buffer stay in view order (events)
        if streams not in (1, 2) or (streams == 2 and compact):
            raise ValueError("streams must be 1 or 2 (2 only without compact)")
        self.n_streams = streams
        self.side = torch.cuda.Stream(device=device) if streams == 2 else None
        # compact: reduce only the union of the ranks' visible particles (VisibleUnionReducer)
        self.reducer = VisibleUnionReducer(params.P, params.flat.shape[0], device) if compact else None
        self.views = views_for_rank(len(self.cameras), rank, world)
        self.group = group
        # sh_factorized: all-gather each view's dL/drgb and rebuild the SH planes
        # (allreduce_grads_sh_factorized); every rank gathers the same number of view
        # slots (the most any rank has), unused slots hold zeros and contribute nothing
        self.drgb = self.cams = None
        if sh_factorized:
            n_slots = -(-len(self.cameras) // max(world, 1))
            self.drgb = torch.zeros((n_slots, 3, params.P), dtype=torch.float32, device=device)
            rows = torch.zeros((n_slots, 12), dtype=torch.float32)
            rows[:, 0] = rows[:, 4] = rows[:, 8] = 1.0
            for j, v in enumerate(self.views):
                c = self.cameras[v]
                rows[j] = torch.tensor([float(x) for x in list(c.R.reshape(9)) + list(c.t.reshape(3))])
            self.cams = rows.to(device)
        self.renderers = {}
        for v in self.views:
            c = self.cameras[v]
            key = (c.width, c.height)
            if key not in self.renderers:
                self.renderers[key] = [Renderer(params.P, c.width, c.height, device=device) for _ in range(streams)]
        self.grads = PlanarParams.zeros(params.P, params.sh_degree, device)
        self.images = {}
        # per view: the frame's (overflow, slots) counters after its forward, copied on the
        # device; read once per step (one host sync instead of one per view)
        self.status = torch.zeros((max(len(self.views), 1), 2), dtype=torch.int64, device=device)

    def _views(self, dL_dimages: dict, main) -> bool:
        """Every view of this rank fwd+bwd (views alternate between `main` and the side
        stream when streams = 2); False (after growing the frames) if a frame overflowed."""
        ctx = (lambda q: torch.cuda.stream(q)) if main is not None else (lambda q: _nullctx())
        first = True
        with ctx(main):
            if self.reducer is not None:
                self.reducer.reset()
            elif self.drgb is not None:
                self.drgb.zero_()
        if self.side is not None:
            self.side.wait_stream(main)
        prev = None  # the previous view's S5b (streams = 2)
        ovf = L.GES_CTR_OVERFLOW
        for j, v in enumerate(self.views):
            cam = self.cameras[v]
            q = self.side if (self.side is not None and j % 2 == 1) else main
            r = self.renderers[(cam.width, cam.height)][j % self.n_streams]
            with ctx(q):
                img = torch.empty((3, cam.height, cam.width), dtype=torch.float32, device=self.grads.flat.device)
                r.forward(self.params, cam, self.settings, img, stream=q, check_overflow=False)
                cnt = r.frame.view("counters", torch.int64, L.GES_CTR_N)
                self.status[j, 0].copy_(cnt[ovf])
                self.status[j, 1].copy_(cnt[L.GES_CTR_SLOTS])
            self.images[v] = img
            if self.reducer is not None:
                self.reducer.add_view(r.frame, q)
            drgb = self.drgb[j] if self.drgb is not None else None
            if self.side is None:
                r.backward(self.params, cam, self.settings, dL_dimages[v], grads=self.grads,
                           accumulate=not first, stream=q, drgb=drgb)
            else:
                ges_render_bwd_tiles(self.settings, r.frame, dL_dimages[v], q)
                if prev is not None:
                    q.wait_event(prev)  # S5b accumulations in view order, never concurrent
                ges_backward_particles(self.params, cam, self.settings, r.frame, self.grads,
                                       accumulate=not first, stream=q, drgb=drgb)
                prev = torch.cuda.Event()
                prev.record(q)
            first = False
        if first:  # no views on this rank: contribute zeros
            with ctx(main):
                self.grads.flat.zero_()
        if self.side is not None:
            main.wait_stream(self.side)
        if not self.views:
            return True
        with ctx(main):  # (the copy is ordered after the views on `main`)
            st = self.status[:len(self.views)].cpu()  # one host sync per step
        if not bool(st[:, 0].any()):
            return True
        keys = {(self.cameras[v].width, self.cameras[v].height) for j, v in enumerate(self.views) if st[j, 0]}
        for key in keys:  # the exact slot count: the next attempt fits unless the scene changed
            for r in self.renderers[key]:
                r.grow(int(st[:, 1].max()))
        return False

    def step(self, dL_dimages: dict, stream=None) -> PlanarParams:
        """dL_dimages: view -> [3][H][W] device tensor, for this rank's views.  Everything
        runs on `stream` (default: torch's current stream); the collectives are issued on
        torch's current stream after it waits for `stream`, and `stream` waits for them."""
        cur = torch.cuda.current_stream() if torch.cuda.is_available() else None
        main = stream if stream is not None else cur
        if stream is not None and cur is not None:
            stream.wait_stream(cur)  # inputs produced on the current stream
        for attempt in range(3):
            if self._views(dL_dimages, main):
                break
            if attempt == 2:
                raise L.GESError("pair capacity still exceeded after regrowing the frames twice")
        if stream is not None and cur is not None:
            cur.wait_stream(stream)  # the masks and gradients are complete before any collective
        if self.reducer is not None:
            self.reducer.allreduce(self.grads.flat, self.group)
        elif self.drgb is not None:
            p = self.params
            allreduce_grads_sh_factorized(
                self.grads.flat, p.sh_degree, self.drgb, self.cams,
                lambda d, c, o: sh_grad_from_colour(p, c, d, out=o), self.group)
        else:
            allreduce_grads(self.grads.flat, self.group)
        if stream is not None and cur is not None:
            stream.wait_stream(cur)
        return self.grads


# ---------------------------------------------------------------------------
# screen-tile bands
# ---------------------------------------------------------------------------
def band_pixel_rows(height: int, rank: int, world: int) -> torch.Tensor:
    """Image rows rendered by `rank`: the 16-row tile rows rank, rank + world, ..."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    tiles_y = (height + TILE - 1) // TILE
    rows = [r * TILE + j for r in range(rank, tiles_y, world) for j in range(TILE) if r * TILE + j < height]
    return torch.tensor(rows, dtype=torch.long)


def band_settings(settings: Settings, rank: int, world: int) -> Settings:
    b, n = (rank, world) if world > 1 else (0, 1)
    return dataclasses.replace(settings, tile_row_begin=b, tile_row_step=n)


def gather_bands(image: torch.Tensor, rank: int, world: int, group=None) -> torch.Tensor:
    """All-gather the band rows of a [3][H][W] image (each rank wrote only its own
    band) into the full image on every rank (one all_gather of equal-size,
    padded band buffers; rows are then scattered back in place)."""
    if world == 1:
        return image
    H = image.shape[1]
    rows = [band_pixel_rows(H, r, world).to(image.device) for r in range(world)]
    n_max = max(int(x.numel()) for x in rows)
    mine = torch.zeros((3, n_max, image.shape[2]), dtype=image.dtype, device=image.device)
    mine[:, :rows[rank].numel()] = image.index_select(1, rows[rank])
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    out = torch.empty_like(image)
    for r in range(world):
        out.index_copy_(1, rows[r], parts[r][:, :rows[r].numel()])
    return out


class BandParallelFrame:
    """This rank's screen-tile band of one frame: forward (gathered image) and
    backward (allreduced parameter gradients)."""

    def __init__(self, params: PlanarParams, camera, settings: Settings, rank: int, world: int, device="cuda",
                 group=None):
        self.params, self.camera, self.rank, self.world, self.group = params, camera, rank, world, group
        self.settings = band_settings(settings, rank, world)
        self.renderer = Renderer(params.P, camera.width, camera.height, device=device)
        self.grads = PlanarParams.zeros(params.P, params.sh_degree, device)

    def forward(self, stream=None) -> torch.Tensor:
        img = self.renderer.forward(self.params, self.camera, self.settings, stream=stream)
        return gather_bands(img, self.rank, self.world, self.group)

    def backward(self, dL_dimage: torch.Tensor, stream=None) -> PlanarParams:
        self.renderer.backward(self.params, self.camera, self.settings, dL_dimage, grads=self.grads, stream=stream)
        allreduce_grads(self.grads.flat, self.group)
        return self.grads
