"""B200-native GES tile rasterizer (arXiv 2402.10128, Generalized Exponential
Splatting): hand-written sm_100a CUDA behind the C ABI of include/ges.h.

There is no CPU fallback: without a built libges.so (and a CUDA device) the
entry points raise.
"""
from ._lib import GESError, load  # noqa: F401
from .api import (PARAM_NAMES, Adam, AdamSettings, DensityControl, DensitySettings, Frame, Loss,  # noqa: F401
                  LossSettings, PlanarParams, Renderer, Settings, c_camera, ges_backward_particles,
                  ges_loss_mask_dims, ges_preprocess, ges_render_bwd, ges_render_bwd_tiles, ges_render_fwd,
                  ges_reset, ges_sort, n_planes, plane_counts, MixSweep, mix_runs, ges_mix_signal,
                  ges_theorem1_errors, MIX_MODELS, reorder, count_nonfinite,
                  camera_rows, sh_grad_from_colour)

__all__ = ["GESError", "load", "Frame", "PlanarParams", "Renderer", "Settings", "ges_preprocess", "ges_sort",
           "ges_render_fwd", "ges_render_bwd", "ges_render_bwd_tiles", "ges_backward_particles", "n_planes",
           "plane_counts", "PARAM_NAMES", "c_camera", "Loss", "LossSettings", "ges_loss_mask_dims",
           "Adam", "AdamSettings", "DensityControl", "DensitySettings", "ges_reset", "MixSweep", "mix_runs",
           "ges_mix_signal", "ges_theorem1_errors", "MIX_MODELS", "reorder", "count_nonfinite",
           "camera_rows", "sh_grad_from_colour"]
