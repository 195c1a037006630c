"""Thin Python binding of the GES C ABI (include/ges.h).

PyTorch is used for device memory, streams and process groups only; every
step of the rasterizer runs in libges.so's sm_100a kernels.  The four entry
points keep the C names (ges_preprocess, ges_sort, ges_render_fwd,
ges_render_bwd); `Renderer` is a convenience owner of one frame workspace.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Optional, Sequence

import torch

from . import _lib as L

PARAM_NAMES = ("mean", "log_scale", "quat", "opacity_logit", "sh", "beta")


def plane_counts(sh_degree: int):
    K = (sh_degree + 1) ** 2
    return {"mean": 3, "log_scale": 3, "quat": 4, "opacity_logit": 1, "sh": 3 * K, "beta": 1}


def n_planes(sh_degree: int) -> int:
    return sum(plane_counts(sh_degree).values())


@dataclasses.dataclass
class Settings:
    rho: float = 0.1                 # PAPER.md:397 "shape strength ... 0.1"
    phi_mode: int = L.GES_PHI_SCALE
    gaussian_only: int = 0
    background: Sequence[float] = (0.0, 0.0, 0.0)
    tile_row_begin: int = 0          # screen-tile band: rows begin + k*step (ges.h)
    tile_row_step: int = 1
    kernel: int = L.GES_KERNEL_PHI_GAUSS  # GES_KERNEL_EXACT_BETA: Eq. 2 per pixel (NEXT-3)

    def c(self) -> L.ges_settings:
        s = L.ges_settings()
        s.rho, s.phi_mode, s.gaussian_only = float(self.rho), int(self.phi_mode), int(self.gaussian_only)
        for k in range(3):
            s.background[k] = float(self.background[k])
        s.tile_row_begin, s.tile_row_step = int(self.tile_row_begin), int(self.tile_row_step)
        s.kernel = int(self.kernel)
        return s


class PlanarParams:
    """Planar SoA fp32 buffer [C][P] (one allocation) with named plane views."""

    def __init__(self, flat: torch.Tensor, P: int, sh_degree: int):
        assert flat.dtype == torch.float32 and flat.is_contiguous() and flat.shape == (n_planes(sh_degree), P)
        self.flat, self.P, self.sh_degree = flat, P, sh_degree
        o = 0
        for n, c in plane_counts(sh_degree).items():
            v = flat[o:o + c]
            setattr(self, n, v[0] if n in ("opacity_logit", "beta") else v)
            o += c

    @classmethod
    def empty(cls, P: int, sh_degree: int, device="cuda", pin_memory=False):
        t = torch.empty((n_planes(sh_degree), P), dtype=torch.float32, device=device, pin_memory=pin_memory)
        return cls(t, P, sh_degree)

    @classmethod
    def zeros(cls, P: int, sh_degree: int, device="cuda"):
        return cls(torch.zeros((n_planes(sh_degree), P), dtype=torch.float32, device=device), P, sh_degree)

    @classmethod
    def from_inputs(cls, parts, device="cuda", pin_memory=False):
        """From a ges_inputs.Particles (numpy planes)."""
        flat = torch.from_numpy(parts.flat())
        if pin_memory:
            flat = flat.pin_memory()
        if device != "cpu":
            flat = flat.to(device)
        return cls(flat.contiguous(), parts.P, parts.sh_degree)

    def c_particles(self) -> L.ges_particles:
        p = L.ges_particles()
        p.P, p.sh_degree = self.P, self.sh_degree
        for n in PARAM_NAMES:
            setattr(p, n, getattr(self, n).data_ptr())
        return p

    def c_grads(self, accumulate: bool, mean2d: Optional[torch.Tensor] = None,
                drgb: Optional[torch.Tensor] = None) -> L.ges_grads:
        """mean2d (optional): a [2][P] fp32 device tensor for dL/d(u, v); drgb (optional): a
        [3][P] one for the view's dL/d rgb (ges.h ges_grads)."""
        g = L.ges_grads()
        for n in PARAM_NAMES:
            setattr(g, n, getattr(self, n).data_ptr())
        if mean2d is not None:
            assert mean2d.dtype == torch.float32 and mean2d.is_contiguous() and mean2d.numel() == 2 * self.P
            g.mean2d = mean2d.data_ptr()
        if drgb is not None:
            assert drgb.dtype == torch.float32 and drgb.is_contiguous() and drgb.numel() == 3 * self.P
            g.drgb = drgb.data_ptr()
        g.accumulate = 1 if accumulate else 0
        return g


def c_camera(cam) -> L.ges_camera:
    """From any object with width, height, fx, fy, cx, cy, near, R (3x3), t (3)."""
    c = L.ges_camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy, c.near_z = cam.fx, cam.fy, cam.cx, cam.cy, cam.near
    R = [float(x) for x in list(cam.R.reshape(9))]
    t = [float(x) for x in list(cam.t.reshape(3))]
    for k in range(9):
        c.R[k] = R[k]
    for k in range(3):
        c.t[k] = t[k]
    return c


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Frame:
    """One frame workspace (a single torch uint8 allocation) and its C struct."""

    # the frame's sub-arrays in carving order (ges.h ges_frame_layout)
    LAYOUT = ("counters", "row_count", "tile_count", "row_pairs", "tile_bucket", "lb_rows", "lb_cols", "depth",
              "pay0", "pay1", "pay2", "pay3", "radius", "rect", "status", "flags", "drgb_ddir", "vis_key0",
              "vis_val0", "vis_key1", "vis_val1", "sorted_vis", "radix_hist", "items", "rowlist", "col_excl", "list",
              "ranges", "final_T", "n_contrib", "tile_order", "grad2d")

    def __init__(self, P: int, width: int, height: int, pair_capacity: int, device="cuda",
                 poison: Optional[int] = None, guard: int = 0):
        """poison (tests): fill the workspace with this byte instead of zeros (grad2d,
        which ges.h requires zeroed, is still zeroed); guard: extra bytes after the
        workspace, filled with the poison byte."""
        lib = L.load()
        nbytes = lib.ges_workspace_bytes(P, width, height, pair_capacity)
        if nbytes == 0:
            raise L.GESError("invalid frame size")
        if poison is None:
            self.ws = torch.zeros(nbytes + 256 + guard, dtype=torch.uint8, device=device)  # zero once (ges.h)
        else:
            self.ws = torch.full((nbytes + 256 + guard,), int(poison), dtype=torch.uint8, device=device)
        base = self.ws.data_ptr()
        self.offset = (-base) % 256
        self.nbytes = nbytes
        self.c = L.ges_frame()
        L.check(lib.ges_frame_init(C.c_void_p(base + self.offset), nbytes, P, width, height, pair_capacity,
                                   C.byref(self.c)), "ges_frame_init")
        self.P, self.width, self.height, self.pair_capacity = P, width, height, pair_capacity
        if poison is not None:
            off, size = self.layout()["grad2d"]
            self.ws[self.offset + off:self.offset + off + size].zero_()

    def layout(self) -> dict:
        """name -> (byte offset from the aligned workspace base, bytes) of every sub-array."""
        n = C.c_int32(0)
        L.load().ges_frame_layout(C.byref(self.c), None, 0, C.byref(n))
        ext = (C.c_int64 * (2 * n.value))()
        L.check(L.load().ges_frame_layout(C.byref(self.c), C.cast(ext, C.c_void_p), n.value, C.byref(n)),
                "ges_frame_layout")
        assert n.value == len(self.LAYOUT), (n.value, len(self.LAYOUT))
        return {k: (ext[2 * i], ext[2 * i + 1]) for i, k in enumerate(self.LAYOUT)}

    # --- typed views into the workspace (tests / diagnostics) ---
    def view(self, field: str, dtype: torch.dtype, count: int, index: Optional[int] = None) -> torch.Tensor:
        ptr = getattr(self.c, field)
        if index is not None:
            ptr = ptr[index]
        off = ptr - self.ws.data_ptr()
        esz = torch.tensor([], dtype=dtype).element_size()
        return self.ws[off:off + count * esz].view(dtype)

    def counts(self, stream=None) -> L.ges_counts:
        out = L.ges_counts()
        L.check(L.load().ges_counts_get(C.byref(self.c), C.byref(out), C.c_void_p(_stream(stream))),
                "ges_counts_get")
        return out

    @property
    def num_tiles(self) -> int:
        return self.c.num_tiles

    def ranges(self):
        return self.view("ranges", torch.int32, self.num_tiles + 1)

    def list(self, M: int):
        return self.view("list", torch.int32, M)


# --- the four C entry points, same names ------------------------------------
def ges_preprocess(particles: PlanarParams, camera, settings: Settings, frame: Frame, stream=None) -> None:
    p, c, s = particles.c_particles(), c_camera(camera), settings.c()
    L.check(L.load().ges_preprocess(C.byref(p), C.byref(c), C.byref(s), C.byref(frame.c), C.c_void_p(_stream(stream))),
            "ges_preprocess")


def ges_sort(frame: Frame, stream=None) -> None:
    L.check(L.load().ges_sort(C.byref(frame.c), C.c_void_p(_stream(stream))), "ges_sort")


def ges_render_fwd(frame: Frame, settings: Settings, image: torch.Tensor, n_eval: Optional[torch.Tensor] = None,
                   stream=None, n_comp: Optional[torch.Tensor] = None) -> None:
    assert image.dtype == torch.float32 and image.is_contiguous() and image.numel() == 3 * frame.width * frame.height
    s = settings.c()
    ne = C.c_void_p(n_eval.data_ptr()) if n_eval is not None else None
    nc = C.c_void_p(n_comp.data_ptr()) if n_comp is not None else None
    L.check(L.load().ges_render_fwd(C.byref(frame.c), C.byref(s), C.c_void_p(image.data_ptr()), ne, nc,
                                    C.c_void_p(_stream(stream))), "ges_render_fwd")


def ges_render_bwd(particles: PlanarParams, camera, settings: Settings, frame: Frame, dL_dimage: torch.Tensor,
                   grads: PlanarParams, accumulate: bool = False, stream=None,
                   mean2d: Optional[torch.Tensor] = None, drgb: Optional[torch.Tensor] = None) -> None:
    assert dL_dimage.dtype == torch.float32 and dL_dimage.is_contiguous()
    p, c, s, g = particles.c_particles(), c_camera(camera), settings.c(), grads.c_grads(accumulate, mean2d, drgb)
    L.check(L.load().ges_render_bwd(C.byref(p), C.byref(c), C.byref(s), C.byref(frame.c),
                                    C.c_void_p(dL_dimage.data_ptr()), C.byref(g), C.c_void_p(_stream(stream))),
            "ges_render_bwd")


def ges_render_bwd_tiles(settings: Settings, frame: Frame, dL_dimage: torch.Tensor, stream=None) -> None:
    assert dL_dimage.dtype == torch.float32 and dL_dimage.is_contiguous()
    s = settings.c()
    L.check(L.load().ges_render_bwd_tiles(C.byref(s), C.byref(frame.c), C.c_void_p(dL_dimage.data_ptr()),
                                          C.c_void_p(_stream(stream))), "ges_render_bwd_tiles")


def ges_backward_particles(particles: PlanarParams, camera, settings: Settings, frame: Frame, grads: PlanarParams,
                           accumulate: bool = False, stream=None, mean2d: Optional[torch.Tensor] = None,
                           drgb: Optional[torch.Tensor] = None) -> None:
    p, c, s, g = particles.c_particles(), c_camera(camera), settings.c(), grads.c_grads(accumulate, mean2d, drgb)
    L.check(L.load().ges_backward_particles(C.byref(p), C.byref(c), C.byref(s), C.byref(frame.c), C.byref(g),
                                            C.c_void_p(_stream(stream))), "ges_backward_particles")


class Renderer:
    """Owns a frame workspace sized for (P, W, H) and grows the pair capacity
    on overflow (one synchronising count read the first time)."""

    def __init__(self, P: int, width: int, height: int, pair_capacity: Optional[int] = None, device="cuda"):
        self.P, self.width, self.height, self.device = P, width, height, device
        cap = pair_capacity or max(1 << 16, 16 * P)
        self.frame = Frame(P, width, height, cap, device)

    def grow(self, M: int) -> None:
        cap = int(M * 1.25) + 1024
        self.frame = Frame(self.P, self.width, self.height, cap, self.device)

    def forward(self, particles: PlanarParams, camera, settings: Settings, image: Optional[torch.Tensor] = None,
                n_eval=None, stream=None, check_overflow: bool = True, n_comp=None) -> torch.Tensor:
        if image is None:
            image = torch.empty((3, self.height, self.width), dtype=torch.float32, device=self.device)
        for attempt in range(3):
            ges_preprocess(particles, camera, settings, self.frame, stream)
            ges_sort(self.frame, stream)
            ges_render_fwd(self.frame, settings, image, n_eval, stream, n_comp)
            if not check_overflow:
                return image
            cnt = self.frame.counts(stream)
            if not cnt.overflow:
                return image
            self.grow(cnt.slots)   # the exact slot count: the next attempt fits unless the scene changed
        raise L.GESError("pair capacity still exceeded after regrowing the frame twice")

    def backward(self, particles: PlanarParams, camera, settings: Settings, dL_dimage: torch.Tensor,
                 grads: Optional[PlanarParams] = None, accumulate: bool = False, stream=None,
                 drgb: Optional[torch.Tensor] = None) -> PlanarParams:
        if grads is None:
            grads = PlanarParams.zeros(particles.P, particles.sh_degree, self.device)
        ges_render_bwd(particles, camera, settings, self.frame, dL_dimage, grads, accumulate, stream, drgb=drgb)
        return grads


# --- loss front end (ges.h ges_loss*) -------------------
@dataclasses.dataclass
class LossSettings:
    lambda_ssim: float = 0.2
    lambda_omega: float = 0.5
    eps_omega: float = 0.5
    downsample: float = 0.2

    def c(self) -> L.ges_loss_settings:
        s = L.ges_loss_settings()
        s.lambda_ssim, s.lambda_omega = float(self.lambda_ssim), float(self.lambda_omega)
        s.eps_omega, s.downsample = float(self.eps_omega), float(self.downsample)
        return s


def ges_loss_mask_dims(width: int, height: int, downsample: float = 0.2):
    wd, hd = C.c_int32(), C.c_int32()
    L.check(L.load().ges_loss_mask_dims(width, height, downsample, C.byref(wd), C.byref(hd)), "ges_loss_mask_dims")
    return int(wd.value), int(hd.value)


class Loss:
    """Owns the loss workspace for one image size (marshalling only: every step
    runs in libges.so's loss kernels)."""

    def __init__(self, width: int, height: int, settings: Optional[LossSettings] = None, device="cuda"):
        self.W, self.H, self.settings = width, height, settings or LossSettings()
        nbytes = L.load().ges_loss_workspace_bytes(width, height, self.settings.downsample)
        if nbytes == 0:
            raise L.GESError("ges_loss_workspace_bytes: invalid size")
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.Wd, self.Hd = ges_loss_mask_dims(width, height, self.settings.downsample)
        self.out = torch.zeros(4, dtype=torch.float32, device=device)

    def mask(self, gt: torch.Tensor, omega: float, mask_lo: Optional[torch.Tensor] = None, stream=None):
        assert gt.dtype == torch.float32 and gt.is_contiguous() and gt.numel() == 3 * self.W * self.H
        if mask_lo is None:
            mask_lo = torch.empty((self.Hd, self.Wd), dtype=torch.uint8, device=self.ws.device)
        s = self.settings.c()
        L.check(L.load().ges_loss_mask(C.c_void_p(gt.data_ptr()), self.W, self.H, float(omega), C.byref(s),
                                       C.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                       C.c_void_p(mask_lo.data_ptr()), C.c_void_p(_stream(stream))), "ges_loss_mask")
        return mask_lo

    def __call__(self, image: torch.Tensor, gt: torch.Tensor, mask_lo: Optional[torch.Tensor],
                 dL_dimage: Optional[torch.Tensor] = None, stream=None):
        """Returns (loss_out[4] = (L, L1, SSIM, L_omega) on the device, dL/dimage)."""
        for t in (image, gt):
            assert t.dtype == torch.float32 and t.is_contiguous() and t.numel() == 3 * self.W * self.H
        if dL_dimage is None:
            dL_dimage = torch.empty_like(image)
        s = self.settings.c()
        mp = C.c_void_p(mask_lo.data_ptr()) if mask_lo is not None else None
        L.check(L.load().ges_loss(C.c_void_p(image.data_ptr()), C.c_void_p(gt.data_ptr()), mp, self.W, self.H,
                                  C.byref(s), C.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                  C.c_void_p(dL_dimage.data_ptr()), C.c_void_p(self.out.data_ptr()),
                                  C.c_void_p(_stream(stream))), "ges_loss")
        return self.out, dL_dimage


# --- optimizer and density control (ges.h ges_adam_step ...) ---
@dataclasses.dataclass
class AdamSettings:
    """Per-group learning rates of PAPER.md:1231-1244 (readings DESIGN.md R29)."""
    lr_pos_init: float = 1.6e-4
    lr_pos_final: float = 1.6e-6
    lr_pos_delay_mult: float = 0.01
    lr_pos_max_steps: int = 30000
    lr_feature: float = 2.5e-3
    lr_opacity: float = 0.05
    lr_scaling: float = 5e-3
    lr_rotation: float = 1e-3
    lr_shape: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15

    def lr_position(self, step: int) -> float:
        return L.load().ges_lr_position(step, self.lr_pos_init, self.lr_pos_final, self.lr_pos_delay_mult,
                                        self.lr_pos_max_steps, 0)

    def c(self, step: int) -> L.ges_adam_settings:
        s = L.ges_adam_settings()
        s.step = int(step)
        s.lr_position = self.lr_position(step)
        s.lr_scaling, s.lr_rotation, s.lr_opacity = self.lr_scaling, self.lr_rotation, self.lr_opacity
        s.lr_feature_dc, s.lr_feature_rest, s.lr_shape = self.lr_feature, self.lr_feature / 20.0, self.lr_shape
        s.beta1, s.beta2, s.eps = self.beta1, self.beta2, self.eps
        return s


class Adam:
    """Fused Adam over a PlanarParams buffer (moments owned here)."""

    def __init__(self, params: PlanarParams, settings: Optional[AdamSettings] = None):
        self.settings = settings or AdamSettings()
        self.m = PlanarParams.zeros(params.P, params.sh_degree, params.flat.device)
        self.v = PlanarParams.zeros(params.P, params.sh_degree, params.flat.device)
        self.t = 0

    def step_range(self, params: PlanarParams, grads_range: torch.Tensor, begin: int, count: int,
                   stream=None) -> None:
        """One step of the flat entries [begin, begin + count) only (ges_adam_step_range: a
        ZeRO-1 shard); grads_range holds their gradients.  Advances the step count."""
        self.t += 1
        s = self.settings.c(self.t)
        assert grads_range.dtype == torch.float32 and grads_range.is_contiguous() and grads_range.numel() >= count
        L.check(L.load().ges_adam_step_range(C.c_void_p(params.flat.data_ptr()), C.c_void_p(grads_range.data_ptr()),
                                             C.c_void_p(self.m.flat.data_ptr()), C.c_void_p(self.v.flat.data_ptr()),
                                             params.P, params.sh_degree, C.byref(s), int(begin), int(count),
                                             C.c_void_p(_stream(stream))), "ges_adam_step_range")

    def step(self, params: PlanarParams, grads: PlanarParams, stream=None) -> None:
        self.t += 1
        s = self.settings.c(self.t)
        L.check(L.load().ges_adam_step(C.c_void_p(params.flat.data_ptr()), C.c_void_p(grads.flat.data_ptr()),
                                       C.c_void_p(self.m.flat.data_ptr()), C.c_void_p(self.v.flat.data_ptr()),
                                       params.P, params.sh_degree, C.byref(s), C.c_void_p(_stream(stream))),
                "ges_adam_step")


def camera_rows(cameras, device="cuda") -> torch.Tensor:
    """[n][12] fp32 (R row-major, then t) of camera objects, as ges_sh_grad_from_colour takes them."""
    rows = [[float(x) for x in list(c.R.reshape(9))] + [float(x) for x in list(c.t.reshape(3))] for c in cameras]
    return torch.tensor(rows, dtype=torch.float32).reshape(len(rows), 12).to(device)


def sh_grad_from_colour(params: PlanarParams, cams: torch.Tensor, drgb: torch.Tensor,
                        out: Optional[torch.Tensor] = None, accumulate: bool = False, stream=None) -> torch.Tensor:
    """The SH gradient [3K][P] of n views from their cameras (cams: [n][12], camera_rows) and
    their per-view dL/d rgb (drgb: [n][3][P], ges_grads.drgb) -- ges_sh_grad_from_colour."""
    n = cams.shape[0]
    assert cams.dtype == torch.float32 and cams.is_contiguous() and cams.shape == (n, 12)
    assert drgb.dtype == torch.float32 and drgb.is_contiguous() and drgb.numel() == 3 * n * params.P
    if out is None:
        out = torch.empty_like(params.sh)
    assert out.dtype == torch.float32 and out.is_contiguous() and out.shape == params.sh.shape
    L.check(L.load().ges_sh_grad_from_colour(C.c_void_p(params.mean.data_ptr()), params.P, params.sh_degree,
                                             C.c_void_p(cams.data_ptr()), n, C.c_void_p(drgb.data_ptr()),
                                             C.c_void_p(out.data_ptr()), 1 if accumulate else 0,
                                             C.c_void_p(_stream(stream))), "ges_sh_grad_from_colour")
    return out


def count_nonfinite(*tensors: torch.Tensor, stream=None) -> torch.Tensor:
    """Failure detection (debug): the number of NaN / Inf values in fp32 device tensors,
    as a device int64 scalar (no synchronisation; `.item()` reads it)."""
    out = torch.zeros(1, dtype=torch.int64, device=tensors[0].device if tensors else "cuda")
    for t in tensors:
        assert t.dtype == torch.float32 and t.is_contiguous() and t.is_cuda
        L.check(L.load().ges_count_nonfinite(C.c_void_p(t.data_ptr()), t.numel(), C.c_void_p(out.data_ptr()),
                                             C.c_void_p(_stream(stream))), "ges_count_nonfinite")
    return out[0]


def reorder(params: PlanarParams, opt: Optional["Adam"] = None, stream=None):
    """Particle storage order (ges_reorder): a new PlanarParams in the Morton order of
    the means, and perm (int32 [P], perm[j] = old index of new particle j).  With an
    Adam `opt`, its moments are permuted alongside (replaced in place).  Call after
    loading a scene and after densify/prune."""
    P, deg, dev = params.P, params.sh_degree, params.flat.device
    lib = L.load()
    nb = lib.ges_reorder_workspace_bytes(P)
    ws = torch.empty(nb + 256, dtype=torch.uint8, device=dev)
    base = ws.data_ptr() + (-ws.data_ptr()) % 256
    out = PlanarParams.empty(P, deg, dev)
    perm = torch.empty(P, dtype=torch.int32, device=dev)
    m_in = m_out = v_in = v_out = None
    if opt is not None:
        m_out, v_out = PlanarParams.empty(P, deg, dev), PlanarParams.empty(P, deg, dev)
        m_in, v_in = C.c_void_p(opt.m.flat.data_ptr()), C.c_void_p(opt.v.flat.data_ptr())
    L.check(lib.ges_reorder(C.c_void_p(params.flat.data_ptr()), C.c_void_p(out.flat.data_ptr()), m_in,
                            C.c_void_p(m_out.flat.data_ptr()) if m_out is not None else None, v_in,
                            C.c_void_p(v_out.flat.data_ptr()) if v_out is not None else None, P, deg,
                            C.c_void_p(perm.data_ptr()), C.c_void_p(base), nb, C.c_void_p(_stream(stream))),
            "ges_reorder")
    if opt is not None:
        opt.m, opt.v = m_out, v_out
    return out, perm


def ges_reset(params: PlanarParams, what: int, stream=None) -> None:
    """what = 0: opacity reset (kappa <= 0.01); 1: shape reset (beta = 2)."""
    L.check(L.load().ges_reset(C.c_void_p(params.flat.data_ptr()), params.P, params.sh_degree, int(what),
                               C.c_void_p(_stream(stream))), "ges_reset")


@dataclasses.dataclass
class DensitySettings:
    grad_threshold: float = 3e-4
    percent_dense: float = 0.01
    scene_extent: float = 1.0
    opacity_prune: float = 0.005
    shape_prune: float = 0.5
    rho: float = 0.1
    seed: int = 0

    def c(self) -> L.ges_density_settings:
        s = L.ges_density_settings()
        s.grad_threshold, s.percent_dense, s.scene_extent = self.grad_threshold, self.percent_dense, self.scene_extent
        s.opacity_prune, s.shape_prune, s.rho, s.seed = self.opacity_prune, self.shape_prune, self.rho, int(self.seed)
        return s


class DensityControl:
    """View-space gradient statistics and the densify/prune pass."""

    def __init__(self, P: int, device="cuda"):
        self.accum = torch.zeros(P, dtype=torch.float32, device=device)
        self.count = torch.zeros(P, dtype=torch.float32, device=device)

    def accumulate(self, frame: Frame, stream=None) -> None:
        """Call between ges_render_bwd_tiles and ges_backward_particles."""
        L.check(L.load().ges_densify_stats(C.byref(frame.c), C.c_void_p(self.accum.data_ptr()),
                                           C.c_void_p(self.count.data_ptr()), C.c_void_p(_stream(stream))),
                "ges_densify_stats")

    def densify_prune(self, params: PlanarParams, opt: Adam, settings: DensitySettings, stream=None,
                      group=None):
        """Returns the new PlanarParams; opt's moments are replaced; the statistics reset (one sync).
        Under torch.distributed (world > 1) the statistics are first summed over `group`
        (dist.allreduce_density_stats), so every data-parallel rank densifies identically."""
        from .dist import allreduce_density_stats
        if stream is not None:  # the collective runs on torch's current stream: order it after `stream`
            cur = torch.cuda.current_stream()
            cur.wait_stream(stream)
            allreduce_density_stats(self.accum, self.count, group)
            stream.wait_stream(cur)
        else:
            allreduce_density_stats(self.accum, self.count, group)
        P, deg, dev = params.P, params.sh_degree, params.flat.device
        cap = 2 * P
        outs = [torch.empty((n_planes(deg), cap), dtype=torch.float32, device=dev) for _ in range(3)]
        ws = torch.empty(L.load().ges_densify_workspace_bytes(P), dtype=torch.uint8, device=dev)
        p_out = torch.zeros(1, dtype=torch.int64, device=dev)
        s = settings.c()
        L.check(L.load().ges_densify_prune(
            C.c_void_p(params.flat.data_ptr()), C.c_void_p(opt.m.flat.data_ptr()), C.c_void_p(opt.v.flat.data_ptr()),
            C.c_void_p(self.accum.data_ptr()), C.c_void_p(self.count.data_ptr()), P, deg, C.byref(s),
            C.c_void_p(outs[0].data_ptr()), C.c_void_p(outs[1].data_ptr()), C.c_void_p(outs[2].data_ptr()), cap,
            C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(p_out.data_ptr()), C.c_void_p(_stream(stream))),
            "ges_densify_prune")
        n = int(p_out.item())
        new = [PlanarParams(o[:, :n].contiguous(), n, deg) for o in outs]
        opt.m, opt.v = new[1], new[2]
        self.accum = torch.zeros(n, dtype=torch.float32, device=dev)
        self.count = torch.zeros(n, dtype=torch.float32, device=dev)
        return new[0]


# ---- NEXT-4: the 1-D mixture simulation and Theorem 1 (include/ges.h) --------------
MIX_MODELS = ("gmm", "dog", "log", "gef")


def _grid(x_lo: float, x_hi: float, n: int) -> L.ges_mix_grid:
    g = L.ges_mix_grid()
    g.x_lo, g.x_hi, g.n = float(x_lo), float(x_hi), int(n)
    return g


def ges_mix_signal(kind: str, width: float, x_lo: float, x_hi: float, n: int, stream=None) -> torch.Tensor:
    """The ground-truth signal `kind` (L.GES_SIGNALS) on the grid, a device [n] tensor."""
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    g = _grid(x_lo, x_hi, n)
    L.check(L.load().ges_mix_signal(L.GES_SIGNALS.index(kind), float(width), C.byref(g), C.c_void_p(y.data_ptr()),
                                    C.c_void_p(_stream(stream))), "ges_mix_signal")
    return y


def mix_runs(specs: Sequence) -> torch.Tensor:
    """Device run table from (model name, positive, n_comp, target row) tuples."""
    rows = [(MIX_MODELS.index(m), int(bool(p)), int(n), int(t)) for (m, p, n, t) in specs]
    return torch.tensor(rows, dtype=torch.int32, device="cuda").reshape(-1, 4)


class MixSweep:
    """A batch of independent 1-D mixture fits (one CTA each) sharing a grid and a
    target table: params / m / v are device [R][stride] tensors."""

    def __init__(self, runs: torch.Tensor, params: torch.Tensor, targets: torch.Tensor, x_lo: float, x_hi: float):
        self.runs = runs.contiguous()
        self.params = params.contiguous()
        self.targets = targets.contiguous()
        self.grid = _grid(x_lo, x_hi, targets.shape[-1])
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.loss = torch.empty(self.runs.shape[0], dtype=torch.float32, device=self.params.device)
        self.t = 0

    def eval(self, grad: bool = True, stream=None):
        g = torch.empty_like(self.params) if grad else None
        L.check(L.load().ges_mix_eval(
            C.c_void_p(self.runs.data_ptr()), self.runs.shape[0], C.c_void_p(self.params.data_ptr()),
            self.params.shape[1], C.byref(self.grid), C.c_void_p(self.targets.data_ptr()),
            C.c_void_p(self.loss.data_ptr()), C.c_void_p(g.data_ptr() if g is not None else 0),
            C.c_void_p(_stream(stream))), "ges_mix_eval")
        return self.loss, g

    def fit(self, steps: int, lr: float = 1e-2, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
            stream=None) -> torch.Tensor:
        a = L.ges_mix_adam()
        a.lr, a.beta1, a.beta2, a.eps = lr, beta1, beta2, eps
        L.check(L.load().ges_mix_fit(
            C.c_void_p(self.runs.data_ptr()), self.runs.shape[0], C.c_void_p(self.params.data_ptr()),
            C.c_void_p(self.m.data_ptr()), C.c_void_p(self.v.data_ptr()), self.params.shape[1], C.byref(self.grid),
            C.c_void_p(self.targets.data_ptr()), C.byref(a), int(steps), int(self.t),
            C.c_void_p(self.loss.data_ptr()), C.c_void_p(_stream(stream))), "ges_mix_fit")
        self.t += int(steps)
        return self.loss


def ges_theorem1_errors(alpha: torch.Tensor, beta: torch.Tensor, A: float = 1.0, L_width: float = 1.0,
                        intervals: int = 4096, stream=None) -> torch.Tensor:
    """E[a][b] of Theorem 1 (square wave, amplitude A, width L) by quadrature on the device."""
    alpha = alpha.contiguous().float()
    beta = beta.contiguous().float()
    E = torch.empty((alpha.numel(), beta.numel()), dtype=torch.float32, device=alpha.device)
    L.check(L.load().ges_theorem1_errors(C.c_void_p(alpha.data_ptr()), alpha.numel(), C.c_void_p(beta.data_ptr()),
                                         beta.numel(), float(A), float(L_width), int(intervals),
                                         C.c_void_p(E.data_ptr()), C.c_void_p(_stream(stream))),
            "ges_theorem1_errors")
    return E
