"""Training losses on B200 (drop-in for ``splatstream.losses``, losses.py:137-228).

``compute_losses`` runs the fused L1 + SSIM kernel (K6) and the opacity
regulariser kernel; scalars are returned as Python floats like the
reference (one device->host read), ``grad_image`` / ``grad_opacity_logit``
stay on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, errors
from ._lib import check, lib, traced
from .rasterizer import P, stream_handle

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2


@dataclass
class LossBreakdown:
    """losses.py:185-195.  The scalars are Python floats; in deferred error
    mode (errors.py) they are read from the device when first used."""

    _SCALARS = ("l1", "ssim_loss", "rendered", "opacity_reg", "total")

    def __init__(self, l1=None, ssim_loss=None, rendered=None, opacity_reg=None, total=None,
                 grad_image=None, grad_opacity_logit=None, resolve=None):
        self._resolve = resolve
        self._vals = None if resolve is not None else dict(
            l1=l1, ssim_loss=ssim_loss, rendered=rendered, opacity_reg=opacity_reg, total=total)
        self.grad_image = grad_image
        self.grad_opacity_logit = grad_opacity_logit

    def _get(self, k):
        if self._vals is None:
            self._vals = self._resolve()
            self._resolve = None
        return self._vals[k]

    l1 = property(lambda self: self._get("l1"))
    ssim_loss = property(lambda self: self._get("ssim_loss"))
    rendered = property(lambda self: self._get("rendered"))
    opacity_reg = property(lambda self: self._get("opacity_reg"))
    total = property(lambda self: self._get("total"))

    def __repr__(self):
        return "LossBreakdown(" + ", ".join(f"{k}={self._get(k)!r}" for k in self._SCALARS) + ")"


def _img(x, dev):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return x.to(device=dev, dtype=torch.float32).contiguous()


def photometric(rendered: torch.Tensor, target: torch.Tensor, lambda_ssim: float,
                grad: torch.Tensor, sums: torch.Tensor, ws: torch.Tensor | None = None):
    """Enqueue K6: grad <- d rendered_loss / d image, sums[0:2] <- (sum|x-y|, sum SSIM)."""
    H, W = int(rendered.shape[0]), int(rendered.shape[1])
    if ws is None:
        ws = torch.empty(int(lib().ss_loss_workspace_bytes(H, W)), dtype=torch.uint8,
                         device=rendered.device)
    check(lib().ss_loss_l1_ssim(H, W, P(rendered), P(target), float(lambda_ssim), P(grad), None,
                                P(sums), P(ws), ws.numel(), stream_handle()), "ss_loss_l1_ssim")
    return ws


@traced("ss.rendered_loss")
def rendered_loss(rendered, target, lambda_ssim: float = 0.2):
    """losses.py:137-154: (1 - l) mean|x - y| + l (1 - SSIM) and its
    analytic gradient w.r.t. the rendered image (K6; float32 device
    gradient).  Returns (loss, grad)."""
    dev = rendered.device if isinstance(rendered, torch.Tensor) else torch.device("cuda")
    x, y = _img(rendered, dev), _img(target, dev)
    if tuple(x.shape) != tuple(y.shape):
        raise ValueError(f"image shapes differ: {tuple(x.shape)} vs {tuple(y.shape)}")
    grad = torch.empty_like(x)
    sums = torch.zeros(_lib.SS_REDUCE_DOUBLES, dtype=torch.float64, device=dev)
    photometric(x, y, lambda_ssim, grad, sums)
    sh = sums[:2].cpu().numpy()
    l1 = float(sh[0]) / x.numel()
    if lambda_ssim != 0.0:
        return (1.0 - lambda_ssim) * l1 + lambda_ssim * (1.0 - float(sh[1]) / x.numel()), grad
    return l1, grad


PSNR_CAP_DB = 100.0


def ssim_metric(a, b) -> float:
    """losses.py:176-182: mean local SSIM over pixels and channels (the K6
    forward's SSIM sum; images of at least 6 x 6 pixels)."""
    dev = a.device if isinstance(a, torch.Tensor) else torch.device("cuda")
    x, y = _img(a, dev), _img(b, dev)
    if x.shape != y.shape or x.dim() != 3 or x.shape[2] != 3:
        raise ValueError(f"image shapes {tuple(x.shape)} and {tuple(y.shape)} must match (H,W,3)")
    sums = torch.zeros(_lib.SS_REDUCE_DOUBLES, dtype=torch.float64, device=dev)
    photometric(x, y, 1.0, torch.empty_like(x), sums)
    return float(sums[1].item()) / x.numel()


def psnr(a, b) -> float:
    """losses.py:112-116: PSNR in dB for [0, 1] images, capped at 100 dB
    (evaluation metric, off the mapping path: a device reduction)."""
    dev = a.device if isinstance(a, torch.Tensor) else torch.device("cuda")
    x, y = _img(a, dev), _img(b, dev)
    if x.shape != y.shape:
        raise ValueError(f"image shapes {tuple(x.shape)} and {tuple(y.shape)} must match")
    mse = float(((x.double() - y.double()) ** 2).mean().item())
    if mse < 1e-10:
        return PSNR_CAP_DB
    return min(PSNR_CAP_DB, 10.0 * float(np.log10(1.0 / mse)))


@traced("ss.compute_losses")
def compute_losses(rendered, target, opacity_logits, lambda_ssim: float = 0.2,
                   lambda_o: float = 0.001) -> LossBreakdown:
    """losses.py:198-228."""
    dev = opacity_logits.device if isinstance(opacity_logits, torch.Tensor) else (
        rendered.device if isinstance(rendered, torch.Tensor) else torch.device("cuda"))
    x = _img(rendered, dev)
    y = _img(target, dev)
    if tuple(x.shape) != tuple(y.shape):
        raise ValueError(f"image shapes differ: {tuple(x.shape)} vs {tuple(y.shape)}")
    logits = _img(opacity_logits, dev).reshape(-1)
    n = int(logits.numel())
    H, W = int(x.shape[0]), int(x.shape[1])
    grad = torch.empty_like(x)
    sums = torch.zeros(_lib.SS_REDUCE_DOUBLES, dtype=torch.float64, device=dev)
    osum = torch.zeros(_lib.SS_REDUCE_DOUBLES, dtype=torch.float64, device=dev)
    photometric(x, y, lambda_ssim, grad, sums)
    g_logit = torch.empty(n, dtype=torch.float32, device=dev)
    check(lib().ss_opacity_reg(n, P(logits), float(lambda_o), P(g_logit), 0, P(osum),
                               stream_handle()), "ss_opacity_reg")
    dsums = torch.cat((sums[:2], osum[:1]))
    npx = H * W * 3

    def resolve():
        sh = dsums.cpu().numpy()  # one host read
        l1 = float(sh[0] / npx)
        ssim_loss = 1.0 - float(sh[1] / npx) if lambda_ssim != 0.0 else 0.0
        rendered_val = (1.0 - lambda_ssim) * l1 + lambda_ssim * ssim_loss
        reg = float(sh[2] / n) if n else 0.0
        return dict(l1=l1, ssim_loss=ssim_loss, rendered=rendered_val, opacity_reg=reg,
                    total=rendered_val + lambda_o * reg)
    if errors.deferred():
        return LossBreakdown(grad_image=grad, grad_opacity_logit=g_logit, resolve=resolve)
    return LossBreakdown(**resolve(), grad_image=grad, grad_opacity_logit=g_logit)


def opacity_reg(opacities):
    """losses.py:157-168 (host helper on activated opacities)."""
    o = np.asarray(opacities, dtype=np.float64)
    n = o.size
    if n == 0:
        return 0.0, np.zeros(0)
    return float(np.mean(np.abs(o))), np.sign(o) / n


def total_loss(rendered: float, opacity: float, lambda_o: float) -> float:
    """losses.py:171-173."""
    return rendered + lambda_o * opacity


def depth_l1(depth: torch.Tensor, target_depth: torch.Tensor, weight: float = 1.0):
    """Builder extension A15: weight * mean |D - D*| over pixels with D* > 0.
    Returns (loss, grad_depth)."""
    H, W = int(depth.shape[0]), int(depth.shape[1])
    dev = depth.device
    tgt = _img(target_depth, dev)
    g = torch.empty((H, W), dtype=torch.float32, device=dev)
    sums = torch.zeros(_lib.SS_REDUCE_DOUBLES, dtype=torch.float64, device=dev)
    check(lib().ss_depth_l1(H, W, P(depth.contiguous()), P(tgt), float(weight), P(g), P(sums),
                            stream_handle()), "ss_depth_l1")
    s = sums[:2].cpu().numpy()
    return float(weight * s[0] / max(s[1], 1.0)), g


_ = ctypes
