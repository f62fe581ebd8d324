"""Densification statistics, clone/split/prune and opacity reset on B200
(drop-in for ``splatstream.densify``, densify.py:25-173).

``densify_and_prune`` is two C-ABI calls: masks + order-preserving scans
(float64 mask math, bit-exact with the reference on the same stored
values), then the compaction that writes survivors, clones and split
children into a new map.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import check, lib, traced
from .core import GaussianMap
from .rasterizer import ParamGrads, P, stream_handle


@dataclass
class DensifyConfig:
    """densify.py:25-39."""

    interval: int = 500
    grad_threshold: float = 0.001
    prune_opacity: float = 0.02
    split_scale_percentile: float = 0.01
    split_children: int = 2
    split_scale_shrink: float = 1.6
    clone_step: float = 0.01

    def __post_init__(self):
        if self.interval < 1:
            raise ValueError("densify interval must be >= 1")
        if self.grad_threshold <= 0 or self.prune_opacity <= 0:
            raise ValueError("densify thresholds must be positive")


@dataclass
class DensifyResult:
    """densify.py:42-50."""

    survivors: torch.Tensor
    n_new: int
    n_cloned: int
    n_split: int
    n_pruned: int


@traced("ss.seed_from_points")
def seed_from_points(points, colors, scene_extent: float = 1.0, device=None):
    """densify.py:53-83 on the GPU: one isotropic primitive per point, scale =
    mean distance to the 3 nearest neighbours in the cloud (exact kNN on a
    cell grid, ss_seed_from_points).  Returns device float32 tensors
    (positions (n,3), rotations (n,4), log_scales (n,3), opacity_logits (n,),
    sh (n,16,3) with only the DC band set)."""
    dev = torch.device(device) if device is not None else (
        points.device if isinstance(points, torch.Tensor) else torch.device("cuda"))

    def f32(a):
        if isinstance(a, torch.Tensor):
            return a.to(device=dev, dtype=torch.float32).reshape(-1, 3).contiguous()
        return torch.as_tensor(np.asarray(a, np.float64).reshape(-1, 3),
                               dtype=torch.float32).to(dev).contiguous()

    pts, col = f32(points), f32(colors)
    n = int(pts.shape[0])
    if col.shape[0] != n:
        raise ValueError("points and colors must have the same length")
    out = dict(positions=torch.empty((n, 3), dtype=torch.float32, device=dev),
               rotations=torch.empty((n, 4), dtype=torch.float32, device=dev),
               log_scales=torch.empty((n, 3), dtype=torch.float32, device=dev),
               opacity_logits=torch.empty(n, dtype=torch.float32, device=dev),
               sh_dc=torch.empty((n, 3), dtype=torch.float32, device=dev))
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(int(lib().ss_seed_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    check(lib().ss_seed_from_points(n, P(pts), P(col), float(scene_extent),
                                    P(out["positions"]), P(out["rotations"]),
                                    P(out["log_scales"]), P(out["opacity_logits"]),
                                    P(out["sh_dc"]), P(bad), P(ws), ws.numel(), stream_handle()),
          "ss_seed_from_points")
    if int(bad.item()):
        raise ValueError("non-finite point in seed cloud")
    sh = torch.zeros((n, 16, 3), dtype=torch.float32, device=dev)
    sh[:, 0, :] = out["sh_dc"]
    return out["positions"], out["rotations"], out["log_scales"], out["opacity_logits"], sh


@traced("ss.accumulate_grad_stats")
def accumulate_grad_stats(gmap: GaussianMap, grads: ParamGrads) -> GaussianMap:
    """densify.py:86-100."""
    if len(grads) != len(gmap):
        raise ValueError(
            f"gradient length {len(grads)} does not match map length {len(gmap)}")
    contrib = grads.contributed.to(torch.uint8).contiguous()
    mp, gr = gmap.ss(), grads.ss()
    check(lib().ss_accumulate_grad_stats(ctypes.byref(mp), ctypes.byref(gr), P(contrib),
                                         stream_handle()), "ss_accumulate_grad_stats")
    return gmap


def densify_count(gmap: GaussianMap, config: DensifyConfig, scene_extent: float):
    """Phase 1: masks and scans.  Returns (workspace, counts (host), mask)."""
    n = len(gmap)
    dev = gmap.device
    ws = torch.empty(int(lib().ss_densify_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    counts = torch.zeros(5, dtype=torch.int64, device=dev)
    mask = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    mp = gmap.ss()
    limit = float(config.split_scale_percentile) * float(scene_extent)
    check(lib().ss_densify_count(ctypes.byref(mp), config.grad_threshold, config.prune_opacity,
                                 limit, P(ws), ws.numel(), P(counts), P(mask), stream_handle()),
          "ss_densify_count")
    return ws, counts.cpu().numpy(), mask[:n]


@traced("ss.densify_and_prune")
def densify_and_prune(gmap: GaussianMap, config: DensifyConfig, scene_extent: float,
                      rng=None, normals=None, extra_planes=()) -> DensifyResult:
    """densify.py:103-173, in place on ``gmap``.

    Split offsets: ``normals`` ((2 n_split, 3)) if given; else, with a numpy
    ``rng``, drawn exactly where the reference draws them
    (``rng.standard_normal``, densify.py:137); else on the device.
    ``extra_planes``: (in, out) float32 per-Gaussian tensors gathered for
    survivors (the engine passes its Adam moments here; resize_for_densify
    is then a no-op)."""
    if config.split_children != 2:
        raise ValueError("the B200 compaction is specialised for split_children=2")
    n = len(gmap)
    dev = gmap.device
    ws, c, _ = densify_count(gmap, config, scene_extent)
    kept, n_cloned, n_split, n_pruned, n_new = (int(v) for v in c)
    seed = 0
    d_normals = None
    if normals is not None:
        d_normals = torch.as_tensor(np.asarray(normals, np.float32)).reshape(-1, 3).to(dev)
        if d_normals.shape[0] != 2 * n_split:
            raise ValueError("normals must have 2 * n_split rows")
    elif n_split and rng is not None and hasattr(rng, "standard_normal"):
        d_normals = torch.as_tensor(rng.standard_normal((n_split * 2, 3)).astype(np.float32),
                                    device=dev)
    else:
        seed = int(np.random.default_rng().integers(0, 2 ** 63 - 1)) if rng is None else int(rng)
    new = GaussianMap(kept + n_new, dev)
    survivors = torch.empty(max(kept, 1), dtype=torch.int64, device=dev)
    nplanes = len(extra_planes)
    pin = (ctypes.c_void_p * max(nplanes, 1))(*[p[0].data_ptr() for p in extra_planes])
    pout = (ctypes.c_void_p * max(nplanes, 1))(*[p[1].data_ptr() for p in extra_planes])
    pk = (ctypes.c_int32 * max(nplanes, 1))(
        *[int(p[0].numel() // max(n, 1)) for p in extra_planes])
    mp, mo = gmap.ss(), new.ss()
    check(lib().ss_densify_apply(ctypes.byref(mp), P(ws), P(d_normals), seed, config.clone_step,
                                 float(np.log(config.split_scale_shrink)), ctypes.byref(mo),
                                 nplanes, pin, pout, pk, P(survivors), stream_handle()),
          "ss_densify_apply")
    for f in GaussianMap.FIELDS:
        setattr(gmap, f, getattr(new, f))
    return DensifyResult(survivors=survivors[:kept], n_new=n_new, n_cloned=n_cloned,
                         n_split=n_split, n_pruned=n_pruned)


def opacity_reset(gmap: GaussianMap, state=None, ceiling: float = 0.01) -> GaussianMap:
    """Builder extension A16 (the reference has none):
    logit <- logit(min(sigma, ceiling)); opacity moments zeroed."""
    m = state.m.get("opacity_logit") if state is not None else None
    v = state.v.get("opacity_logit") if state is not None else None
    mp = gmap.ss()
    check(lib().ss_opacity_reset(ctypes.byref(mp), float(ceiling), P(m), P(v), stream_handle()),
          "ss_opacity_reset")
    return gmap
