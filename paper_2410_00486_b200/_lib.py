"""ctypes binding of libss_b200.so (include/splatstream_b200.h).

The product path has no CPU fallback: if the CUDA library is missing or no
CUDA device is present, every operator raises.  The library is built
in-tree by ``__graft_entry__.build()`` (``make -C paper_2410_00486_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libss_b200.so")
CSRC = os.path.join(HERE, "csrc")

SS_OK, SS_EINVAL, SS_ECUDA, SS_ECAPACITY = 0, -1, -2, -3
SS_REDUCE_DOUBLES = 2 + 2 * 592
ABI_VERSION = 2

VP = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F32 = ctypes.c_float
F64 = ctypes.c_double
SZ = ctypes.c_size_t


class SSStatus(ctypes.Structure):
    _fields_ = [("first_nonfinite_param", I64), ("first_zero_quat", I64),
                ("first_nonfinite_grad", I64), ("pair_count", I64), ("pair_overflow", I64),
                ("bucket_count", I64), ("visible_count", I64), ("reserved", I64),
                ("opacity_sum", F64), ("reserved2", I64)]


ORDER_MAX_TILES = 16384  # SS_ORDER_MAX_TILES
SS_BWD_SKIP_CLEAR = 1  # ss_backward_splat_ex flag: rows cleared by ss_backward_clear
STATUS_WORDS = 10  # 80-byte ss_status as int64 words (word 8 holds a double)
SNAPSHOT_DOUBLES = 11  # ss_step_snapshot row: 8 status words, opacity sum, 2 loss sums
SN_OPACITY_SUM, SN_L1_SUM, SN_SSIM_SUM = 8, 9, 10
ST_BAD_PARAM, ST_ZERO_QUAT, ST_BAD_GRAD, ST_PAIRS, ST_OVERFLOW, ST_BUCKETS, ST_VISIBLE = range(7)
INT64_MAX = (1 << 63) - 1


class SSMap(ctypes.Structure):
    _fields_ = [("n", I64), ("d_positions", VP), ("d_rotations", VP), ("d_log_scales", VP),
                ("d_opacity_logits", VP), ("d_sh_dc", VP), ("d_sh_rest", VP),
                ("d_grad2d_accum", VP), ("d_grad3d_accum", VP), ("d_obs_count", VP)]


class SSCamera(ctypes.Structure):
    _fields_ = [("fx", F32), ("fy", F32), ("cx", F32), ("cy", F32), ("width", I32),
                ("height", I32), ("R", F32 * 9), ("t", F32 * 3), ("center", F32 * 3)]


class SSRasterOpts(ctypes.Structure):
    _fields_ = [("tile_size", I32), ("bucket_size", I32), ("t_min", F32), ("alpha_min", F32),
                ("alpha_max", F32), ("background", F32 * 3), ("sh_degree", I32),
                ("near_plane", F32), ("dilation", F32), ("with_depth", I32)]


class SSSplats(ctypes.Structure):
    _fields_ = [("d_rec", VP), ("d_depth_key", VP), ("d_tiles", VP), ("d_rect", VP),
                ("d_flags", VP), ("d_aux", VP)]


class SSBins(ctypes.Structure):
    _fields_ = [("pair_capacity", I64), ("d_pair_splat", VP), ("d_tile_start", VP),
                ("d_tile_end", VP), ("d_ckpt_base", VP), ("d_tile_order", VP),
                ("d_tile_cost", VP)]


class SSParamGrads(ctypes.Structure):
    _fields_ = [("d_position", VP), ("d_rotation", VP), ("d_log_scale", VP), ("d_opacity", VP),
                ("d_sh_dc", VP), ("d_sh_rest", VP), ("d_pos2d_norm", VP), ("d_stat_g2d", VP),
                ("d_stat_g3d", VP), ("d_stat_cnt", VP)]


SS_CHAIN_STATS, SS_CHAIN_ACCUMULATE, SS_CHAIN_STAT_PLANES = 1, 2, 4


class SSAdamHP(ctypes.Structure):
    _fields_ = [("lr_position", F32), ("lr_rotation", F32), ("lr_log_scale", F32),
                ("lr_opacity", F32), ("lr_sh_dc", F32), ("lr_sh_rest", F32), ("beta1", F32),
                ("beta2", F32), ("eps", F32), ("bias1", F32), ("bias2", F32),
                ("update_sh_rest", I32)]


P = ctypes.POINTER

_SIGS = {
    "ss_abi_version": (I32, []),
    "ss_status_reset": (I32, [VP, VP]),
    "ss_status_begin_step": (I32, [VP, VP]),
    "ss_status_flags": (I32, [VP, VP, VP]),
    "ss_resize_moments": (I32, [I64, VP, I64, I32, VP, VP, VP, VP]),
    "ss_check_finite": (I32, [I32, VP, VP, VP, VP]),
    "ss_splats_from_projection": (I32, [I64, VP, VP, VP, P(SSCamera), P(SSSplats), VP]),
    "ss_contributed_from_masks": (I32, [P(SSCamera), P(SSBins), VP, VP, VP, VP, I64, VP, I64, VP,
                                        VP]),
    "ss_replay_pixel_states": (I32, [P(SSCamera), P(SSRasterOpts), P(SSSplats), P(SSBins), VP,
                                     VP, VP, VP, I32, I32, I32, VP, VP]),
    "ss_step_snapshot": (I32, [VP, VP, VP, VP]),
    "ss_apply_stat_planes": (I32, [P(SSMap), P(SSParamGrads), VP]),
    "ss_preprocess": (I32, [P(SSMap), P(SSCamera), VP, P(SSRasterOpts), P(SSSplats), VP, VP]),
    "ss_bin_workspace_bytes": (SZ, [I64, I64, I32]),
    "ss_bin_sort": (I32, [I64, P(SSSplats), P(SSCamera), P(SSBins), VP, SZ, VP, VP]),
    "ss_tile_order": (I32, [P(SSCamera), P(SSBins), VP]),
    "ss_blend_forward": (I32, [P(SSCamera), P(SSRasterOpts), P(SSSplats), P(SSBins), VP, VP, VP,
                               VP, VP, VP, VP, VP, VP, VP, I64, VP, VP]),
    "ss_loss_workspace_bytes": (SZ, [I32, I32]),
    "ss_loss_l1_ssim": (I32, [I32, I32, VP, VP, F32, VP, VP, VP, VP, SZ, VP]),
    "ss_opacity_reg": (I32, [I64, VP, F32, VP, I32, VP, VP]),
    "ss_depth_l1": (I32, [I32, I32, VP, VP, F32, VP, VP, VP]),
    "ss_backward_splat": (I32, [P(SSCamera), P(SSRasterOpts), P(SSSplats), P(SSBins), VP, VP,
                                VP, VP, VP, VP, VP, VP, VP, VP, VP, I64, I64, VP, VP, VP, VP]),
    "ss_backward_clear": (I32, [I64, I32, VP, VP, VP, VP]),
    "ss_backward_splat_ex": (I32, [P(SSCamera), P(SSRasterOpts), P(SSSplats), P(SSBins), VP, VP,
                                   VP, VP, VP, VP, VP, VP, VP, VP, VP, I64, I64, VP, VP, VP, I32,
                                   VP]),
    "ss_backward_pixel": (I32, [VP, VP, VP, VP, VP, VP, VP, VP, I64, VP, VP]),
    "ss_seed_workspace_bytes": (SZ, [I64]),
    "ss_seed_from_points": (I32, [I64, VP, VP, F32, VP, VP, VP, VP, VP, VP, VP, SZ, VP]),
    "ss_backward_schedule": (I32, [VP, VP, VP, I64, VP, VP]),
    "ss_chain_backward": (I32, [P(SSMap), P(SSCamera), P(SSRasterOpts), VP, VP, VP, F32, I32,
                                P(SSParamGrads), VP, VP]),
    "ss_adam_step": (I32, [P(SSMap), P(SSParamGrads), P(SSParamGrads), P(SSParamGrads),
                           P(SSAdamHP), VP, VP]),
    "ss_chain_adam": (I32, [P(SSMap), P(SSCamera), VP, P(SSRasterOpts), VP, VP, VP, F32,
                            P(SSParamGrads), P(SSParamGrads), P(SSAdamHP), VP, VP, VP]),
    "ss_accumulate_grad_stats": (I32, [P(SSMap), P(SSParamGrads), VP, VP]),
    "ss_densify_workspace_bytes": (SZ, [I64]),
    "ss_densify_count": (I32, [P(SSMap), F32, F32, F64, VP, SZ, VP, VP, VP]),
    "ss_densify_apply": (I32, [P(SSMap), VP, VP, ctypes.c_uint64, F32, F32, P(SSMap), I32,
                               VP, VP, VP, VP, VP]),
    "ss_opacity_reset": (I32, [P(SSMap), F32, VP, VP, VP]),
}

_lib = None


def _build():
    subprocess.run(["make", "-s", "-C", CSRC, "-j8"], check=True)


def lib():
    """Load the CUDA library (building it in-tree if only the sources exist)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if os.path.exists("/usr/local/cuda/bin/nvcc"):
            _build()
        else:
            raise RuntimeError(f"CUDA extension {LIB_PATH} is missing; run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.ss_abi_version() != ABI_VERSION:
        raise RuntimeError("libss_b200.so ABI version mismatch; rebuild")
    _lib = L
    return L


def check(rc: int, what: str):
    if rc == SS_OK:
        return
    kind = {SS_EINVAL: "invalid argument", SS_ECUDA: "CUDA error",
            SS_ECAPACITY: "workspace too small"}.get(rc, f"error {rc}")
    raise RuntimeError(f"{what} failed: {kind}")


def exported_symbols():
    return list(_SIGS)


def traced(name: str):
    """NVTX range around an API call (nsys / ncu --nvtx timelines show the
    mapping path's stages; a no-op cost without a profiler attached)."""
    import functools

    import torch

    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*a, **k):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*a, **k)
            finally:
                torch.cuda.nvtx.range_pop()
        return wrapper
    return deco
