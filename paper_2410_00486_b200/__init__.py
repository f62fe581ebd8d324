"""B200-native CaRtGS mapping hot path (arxiv 2410.00486).

Drop-in for the mapping path of the reference package ``splatstream``:
the same render / loss / optimise API names (``__init__.py:45-79`` and
``rasterizer/__init__.py:21-36`` of the reference), computing in
hand-written sm_100a kernels (libss_b200.so, C ABI in
include/splatstream_b200.h).  There is no CPU fallback: operators raise if
the CUDA library or device is missing.
"""

from .core import Camera, GaussianMap, logistic, logit
from .densify import (DensifyConfig, DensifyResult, accumulate_grad_stats, densify_and_prune,
                      opacity_reset, seed_from_points)
from .engine import EngineConfig, MappingEngine
from .errors import check_errors, error_mode, set_error_mode
from .losses import (LossBreakdown, compute_losses, depth_l1, opacity_reg, psnr, rendered_loss,
                     ssim_metric, total_loss)
from .optimizer import AdamState, LearningRates, adam_step, resize_for_densify
from .rasterizer import (ParamGrads, Projection, RasterOpts, RenderOutput, TileIndex,
                         backward_pixelwise, backward_splatwise, build_tile_index, chain_backward,
                         project_map, rasterize_forward, render_trajectory, replay_pixel_states,
                         screen_space_grads, screen_space_grads_pixelwise)
from .mapio import load_map, save_map
from .scheduler import KeyframeScheduler, ScheduledMapper
from .scene import CONFIGS, survey_camera, survey_scene

__version__ = "0.1.0"

__all__ = [
    "AdamState", "Camera", "CONFIGS", "DensifyConfig", "DensifyResult", "EngineConfig",
    "GaussianMap", "LearningRates", "LossBreakdown", "MappingEngine", "ParamGrads", "Projection",
    "RasterOpts", "RenderOutput", "TileIndex", "accumulate_grad_stats", "adam_step",
    "backward_pixelwise", "backward_splatwise", "build_tile_index", "chain_backward",
    "check_errors", "compute_losses", "error_mode", "set_error_mode", "densify_and_prune", "depth_l1", "logistic", "logit",
    "KeyframeScheduler", "ScheduledMapper", "load_map", "opacity_reg", "opacity_reset", "psnr",
    "project_map", "rasterize_forward", "render_trajectory", "rendered_loss",
    "replay_pixel_states", "resize_for_densify", "save_map",
    "seed_from_points",
    "ssim_metric",
    "screen_space_grads", "screen_space_grads_pixelwise", "survey_camera", "survey_scene", "total_loss",
]
