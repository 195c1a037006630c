"""ctypes binding of the C ABI in include/ges.h (argument marshalling only).

Every step of the path runs in libges.so's CUDA kernels; this module only
mirrors the C structs.  Importing it on a machine without the built library
raises immediately -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))
# GES_LIB: load an experiment variant built by `_build.py --variant` instead
LIB_PATH = os.environ.get("GES_LIB") or os.path.join(_HERE, "libges.so")

GES_OK, GES_ERR_INVALID_ARG, GES_ERR_CAPACITY, GES_ERR_CUDA, GES_ERR_UNSUPPORTED = range(5)
GES_PHI_SCALE, GES_PHI_VARIANCE = 0, 1
GES_KERNEL_PHI_GAUSS, GES_KERNEL_EXACT_BETA = 0, 1
GES_VISIBLE, GES_CULL_NEAR, GES_DEGENERATE, GES_OFFSCREEN = range(4)
GES_CTR_VISIBLE, GES_CTR_PAIRS, GES_CTR_OVERFLOW, GES_CTR_SLOTS = 0, 1, 2, 3
GES_CTR_TICKET, GES_CTR_TICKET_COLS, GES_CTR_TICKET_EMIT = 4, 5, 6
GES_CTR_KEYMAX, GES_CTR_CULLED_NEAR, GES_CTR_DEGENERATE, GES_CTR_OFFSCREEN, GES_CTR_N = 7, 8, 9, 10, 24

_fp = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)


class ges_particles(C.Structure):
    _fields_ = [("P", C.c_int64), ("sh_degree", C.c_int32), ("_pad", C.c_int32)] + [
        (n, C.c_void_p) for n in ("mean", "log_scale", "quat", "opacity_logit", "sh", "beta")]


class ges_camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("near_z", C.c_float), ("R", C.c_float * 9),
                ("t", C.c_float * 3)]


class ges_settings(C.Structure):
    _fields_ = [("rho", C.c_float), ("phi_mode", C.c_int32), ("gaussian_only", C.c_int32),
                ("background", C.c_float * 3), ("tile_row_begin", C.c_int32), ("tile_row_step", C.c_int32),
                ("kernel", C.c_int32)]


class ges_grads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("mean", "log_scale", "quat", "opacity_logit", "sh", "beta", "mean2d",
                                          "drgb")] + [
        ("accumulate", C.c_int32), ("_pad", C.c_int32)]


class ges_counts(C.Structure):
    _fields_ = [("visible", C.c_int64), ("pairs", C.c_int64), ("slots", C.c_int64), ("capacity", C.c_int64),
                ("culled_near", C.c_int64), ("degenerate", C.c_int64), ("offscreen", C.c_int64),
                ("overflow", C.c_int32), ("_pad", C.c_int32)]


class ges_frame(C.Structure):
    _fields_ = [
        ("P", C.c_int64), ("pair_capacity", C.c_int64),
        ("width", C.c_int32), ("height", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
        ("num_tiles", C.c_int32), ("tile_bits", C.c_int32), ("sh_degree_max", C.c_int32), ("kernel", C.c_int32),
        ("band_begin", C.c_int32), ("band_step", C.c_int32), ("band_rows", C.c_int32), ("depth_key_base", C.c_uint32),
        ("depth", C.c_void_p), ("pay0", C.c_void_p), ("pay1", C.c_void_p), ("pay2", C.c_void_p), ("pay3", C.c_void_p),
        ("radius", C.c_void_p), ("rect", C.c_void_p), ("status", C.c_void_p), ("flags", C.c_void_p),
        ("drgb_ddir", C.c_void_p),
        ("vis_key", C.c_void_p * 2), ("vis_val", C.c_void_p * 2), ("sorted_vis", C.c_void_p),
        ("radix_hist", C.c_void_p), ("items", C.c_void_p), ("row_count", C.c_void_p), ("rowlist", C.c_void_p),
        ("tile_count", C.c_void_p), ("row_pairs", C.c_void_p), ("tile_bucket", C.c_void_p), ("lb_rows", C.c_void_p), ("lb_cols", C.c_void_p),
        ("col_excl", C.c_void_p), ("row_chunks", C.c_int64), ("col_chunks", C.c_int64),
        ("list", C.c_void_p), ("ranges", C.c_void_p),
        ("counters", C.c_void_p), ("zero_bytes", C.c_size_t),
        ("final_T", C.c_void_p), ("n_contrib", C.c_void_p), ("tile_order", C.c_void_p), ("grad2d", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
    ]


class ges_loss_settings(C.Structure):
    _fields_ = [("lambda_ssim", C.c_float), ("lambda_omega", C.c_float), ("eps_omega", C.c_float),
                ("downsample", C.c_float)]


class ges_adam_settings(C.Structure):
    _fields_ = [("step", C.c_int32)] + [(n, C.c_float) for n in (
        "lr_position", "lr_scaling", "lr_rotation", "lr_opacity", "lr_feature_dc", "lr_feature_rest", "lr_shape",
        "beta1", "beta2", "eps")]


class ges_mix_run(C.Structure):
    _fields_ = [("model", C.c_int32), ("positive", C.c_int32), ("n_comp", C.c_int32), ("target", C.c_int32)]


class ges_mix_grid(C.Structure):
    _fields_ = [("x_lo", C.c_float), ("x_hi", C.c_float), ("n", C.c_int32)]


class ges_mix_adam(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]


GES_MIX_GMM, GES_MIX_DOG, GES_MIX_LOG, GES_MIX_GEF = range(4)
GES_MIX_MAX_N, GES_MIX_MAX_SAMPLES = 128, 49152
GES_SIGNALS = ("square", "triangle", "parabolic", "half_sinusoid", "exponential", "gaussian")


class ges_density_settings(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("grad_threshold", "percent_dense", "scene_extent", "opacity_prune",
                                         "shape_prune", "rho")] + [("seed", C.c_uint64)]


EXPORTS = ["ges_workspace_bytes", "ges_frame_init", "ges_frame_layout", "ges_preprocess", "ges_sort", "ges_render_fwd",
           "ges_render_bwd", "ges_render_bwd_tiles", "ges_backward_particles", "ges_counts_get",
           "ges_status_string", "ges_version", "ges_loss_mask_dims", "ges_loss_workspace_bytes", "ges_loss_mask",
           "ges_loss", "ges_lr_position", "ges_adam_step", "ges_adam_step_range", "ges_reset", "ges_densify_stats",
           "ges_densify_workspace_bytes", "ges_densify_prune", "ges_mix_signal", "ges_mix_eval", "ges_mix_fit",
           "ges_theorem1_errors", "ges_probe_mufu", "ges_mask_visible", "ges_grad_pack_workspace_bytes",
           "ges_grad_index", "ges_grad_pack", "ges_grad_unpack", "ges_reorder_workspace_bytes", "ges_reorder",
           "ges_count_nonfinite", "ges_sh_grad_from_colour"]

_lib = None


class GESError(RuntimeError):
    pass


def load(build_if_missing: bool = True) -> C.CDLL:
    """Loads libges.so (building it first if the sources are newer)."""
    global _lib
    if _lib is None:
        if build_if_missing and not os.environ.get("GES_LIB"):
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise GESError(f"libges.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.ges_workspace_bytes.restype = C.c_size_t
        L.ges_workspace_bytes.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int64]
        L.ges_frame_init.restype = C.c_int
        L.ges_frame_init.argtypes = [C.c_void_p, C.c_size_t, C.c_int64, C.c_int32, C.c_int32, C.c_int64,
                                     C.POINTER(ges_frame)]
        L.ges_frame_layout.restype = C.c_int
        L.ges_frame_layout.argtypes = [C.POINTER(ges_frame), C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]
        L.ges_preprocess.restype = C.c_int
        L.ges_preprocess.argtypes = [C.POINTER(ges_particles), C.POINTER(ges_camera), C.POINTER(ges_settings),
                                     C.POINTER(ges_frame), C.c_void_p]
        L.ges_sort.restype = C.c_int
        L.ges_sort.argtypes = [C.POINTER(ges_frame), C.c_void_p]
        L.ges_render_fwd.restype = C.c_int
        L.ges_render_fwd.argtypes = [C.POINTER(ges_frame), C.POINTER(ges_settings), C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p]
        L.ges_render_bwd.restype = C.c_int
        L.ges_render_bwd.argtypes = [C.POINTER(ges_particles), C.POINTER(ges_camera), C.POINTER(ges_settings),
                                     C.POINTER(ges_frame), C.c_void_p, C.POINTER(ges_grads), C.c_void_p]
        L.ges_render_bwd_tiles.restype = C.c_int
        L.ges_render_bwd_tiles.argtypes = [C.POINTER(ges_settings), C.POINTER(ges_frame), C.c_void_p, C.c_void_p]
        L.ges_backward_particles.restype = C.c_int
        L.ges_backward_particles.argtypes = [C.POINTER(ges_particles), C.POINTER(ges_camera), C.POINTER(ges_settings),
                                             C.POINTER(ges_frame), C.POINTER(ges_grads), C.c_void_p]
        L.ges_counts_get.restype = C.c_int
        L.ges_counts_get.argtypes = [C.POINTER(ges_frame), C.POINTER(ges_counts), C.c_void_p]
        L.ges_status_string.restype = C.c_char_p
        L.ges_status_string.argtypes = [C.c_int]
        L.ges_version.restype = C.c_char_p
        L.ges_lr_position.restype = C.c_double
        L.ges_lr_position.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64]
        L.ges_adam_step.restype = C.c_int
        L.ges_adam_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                    C.POINTER(ges_adam_settings), C.c_void_p]
        L.ges_adam_step_range.restype = C.c_int
        L.ges_adam_step_range.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                          C.POINTER(ges_adam_settings), C.c_int64, C.c_int64, C.c_void_p]
        L.ges_reorder_workspace_bytes.restype = C.c_size_t
        L.ges_reorder_workspace_bytes.argtypes = [C.c_int64]
        L.ges_reorder.restype = C.c_int
        L.ges_reorder.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                  C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.ges_reset.restype = C.c_int
        L.ges_reset.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p]
        L.ges_densify_stats.restype = C.c_int
        L.ges_densify_stats.argtypes = [C.POINTER(ges_frame), C.c_void_p, C.c_void_p, C.c_void_p]
        L.ges_densify_workspace_bytes.restype = C.c_size_t
        L.ges_densify_workspace_bytes.argtypes = [C.c_int64]
        L.ges_densify_prune.restype = C.c_int
        L.ges_densify_prune.argtypes = [C.c_void_p] * 5 + [C.c_int64, C.c_int32, C.POINTER(ges_density_settings)] + [
            C.c_void_p] * 3 + [C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
        L.ges_loss_mask_dims.restype = C.c_int
        L.ges_loss_mask_dims.argtypes = [C.c_int32, C.c_int32, C.c_float, C.POINTER(C.c_int32),
                                         C.POINTER(C.c_int32)]
        L.ges_loss_workspace_bytes.restype = C.c_size_t
        L.ges_loss_workspace_bytes.argtypes = [C.c_int32, C.c_int32, C.c_float]
        L.ges_loss_mask.restype = C.c_int
        L.ges_loss_mask.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_float, C.POINTER(ges_loss_settings),
                                    C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
        L.ges_loss.restype = C.c_int
        L.ges_loss.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                               C.POINTER(ges_loss_settings), C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                               C.c_void_p]
        L.ges_mix_signal.restype = C.c_int
        L.ges_mix_signal.argtypes = [C.c_int32, C.c_float, C.POINTER(ges_mix_grid), C.c_void_p, C.c_void_p]
        L.ges_mix_eval.restype = C.c_int
        L.ges_mix_eval.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.POINTER(ges_mix_grid), C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
        L.ges_mix_fit.restype = C.c_int
        L.ges_mix_fit.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.POINTER(ges_mix_grid), C.c_void_p, C.POINTER(ges_mix_adam), C.c_int32, C.c_int32,
                                  C.c_void_p, C.c_void_p]
        L.ges_theorem1_errors.restype = C.c_int
        L.ges_theorem1_errors.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_float, C.c_float,
                                          C.c_int32, C.c_void_p, C.c_void_p]
        L.ges_mask_visible.restype = C.c_int
        L.ges_mask_visible.argtypes = [C.POINTER(ges_frame), C.c_void_p, C.c_void_p]
        L.ges_count_nonfinite.restype = C.c_int
        L.ges_count_nonfinite.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.ges_sh_grad_from_colour.restype = C.c_int
        L.ges_sh_grad_from_colour.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                              C.c_void_p, C.c_int32, C.c_void_p]
        L.ges_grad_pack_workspace_bytes.restype = C.c_size_t
        L.ges_grad_pack_workspace_bytes.argtypes = [C.c_int64]
        L.ges_grad_index.restype = C.c_int
        L.ges_grad_index.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                     C.c_void_p]
        L.ges_grad_pack.restype = C.c_int
        L.ges_grad_pack.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ges_grad_unpack.restype = C.c_int
        L.ges_grad_unpack.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
        L.ges_probe_mufu.restype = C.c_int
        L.ges_probe_mufu.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != GES_OK:
        msg = load().ges_status_string(status).decode()
        raise GESError(f"{what} failed: {msg} ({status})")
