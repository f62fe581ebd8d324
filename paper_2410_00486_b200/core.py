"""Device-resident scene types with the reference's names.

``GaussianMap`` mirrors ``splatstream.core.GaussianMap`` (core.py:110-241):
same field names and pre-activation parameterisation (logit opacity, log
scales), stored as float32 structure-of-arrays on the GPU.  SH
coefficients are kept as the optimizer's two views (optimizer.py:79-87):
``sh_dc`` (N, 3) and ``sh_rest`` (N, 45); ``sh`` reassembles (N, 16, 3).
``Camera`` mirrors ``splatstream.core.Camera`` (core.py:244-301).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .scene import looking_at as _looking_at

SH_COEFFS = 16


def _dev(device=None):
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2410_00486_b200 needs a CUDA device (B200); no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def logistic(x):
    """core.py:16-24 (host helper)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out if out.ndim else float(out)


def logit(p):
    """core.py:27-31."""
    p = np.asarray(p, dtype=np.float64)
    out = np.log(p) - np.log1p(-p)
    return out if out.ndim else float(out)


@dataclass
class Camera:
    """Pinhole camera, x_cam = R x_world + t (core.py:244-301)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray = field(default_factory=lambda: np.eye(3))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.R = np.asarray(self.R, dtype=np.float64).reshape(3, 3)
        self.t = np.asarray(self.t, dtype=np.float64).reshape(3)
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError("focal lengths must be positive")
        if not (0 < self.cx < self.width and 0 < self.cy < self.height):
            raise ValueError("principal point outside image")
        if np.linalg.norm(self.R.T @ self.R - np.eye(3)) >= 1e-6:
            raise ValueError("camera rotation is not orthonormal")

    @property
    def center(self) -> np.ndarray:
        return -self.R.T @ self.t

    @classmethod
    def looking_at(cls, fx, fy, cx, cy, width, height, eye, target, up=(0.0, 1.0, 0.0)):
        c = _looking_at(fx, fy, cx, cy, width, height, eye, target, up)
        return cls(c.fx, c.fy, c.cx, c.cy, c.width, c.height, R=c.R, t=c.t)

    @classmethod
    def of(cls, cam) -> "Camera":
        """Adopt any object with the reference camera's fields."""
        if isinstance(cam, Camera):
            return cam
        return cls(cam.fx, cam.fy, cam.cx, cam.cy, int(cam.width), int(cam.height),
                   R=np.asarray(cam.R), t=np.asarray(cam.t))

    def to_ss(self) -> _lib.SSCamera:
        c = _lib.SSCamera()
        c.fx, c.fy, c.cx, c.cy = self.fx, self.fy, self.cx, self.cy
        c.width, c.height = int(self.width), int(self.height)
        c.R[:] = [float(v) for v in self.R.reshape(9)]
        c.t[:] = [float(v) for v in self.t]
        c.center[:] = [float(v) for v in self.center]
        return c

    @property
    def tiles(self):
        return (self.width + 15) // 16, (self.height + 15) // 16


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


class GaussianMap:
    """Float32 SoA Gaussian store on one CUDA device."""

    FIELDS = ("positions", "rotations", "log_scales", "opacity_logits", "sh_dc", "sh_rest",
              "grad2d_accum", "grad3d_accum", "obs_count")

    def __init__(self, n: int = 0, device=None):
        dev = _dev(device)
        f = dict(dtype=torch.float32, device=dev)
        self.positions = torch.zeros((n, 3), **f)
        self.rotations = torch.zeros((n, 4), **f)
        self.log_scales = torch.zeros((n, 3), **f)
        self.opacity_logits = torch.zeros(n, **f)
        self.sh_dc = torch.zeros((n, 3), **f)
        self.sh_rest = torch.zeros((n, 45), **f)
        self.grad2d_accum = torch.zeros(n, **f)
        self.grad3d_accum = torch.zeros((n, 3), **f)
        self.obs_count = torch.zeros(n, dtype=torch.int32, device=dev)

    @property
    def device(self):
        return self.positions.device

    def __len__(self) -> int:
        return int(self.positions.shape[0])

    @classmethod
    def from_arrays(cls, positions, rotations, log_scales, opacity_logits, sh,
                    device=None) -> "GaussianMap":
        """core.py:150-153.  sh: (N, 16, 3) coefficient-major (or (N, 48))."""
        pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
        n = pos.shape[0]
        g = cls(0, device)
        sh = np.asarray(sh, dtype=np.float64).reshape(n, SH_COEFFS, 3)
        dev = g.device

        def t(a, shape):
            return torch.as_tensor(np.ascontiguousarray(np.asarray(a, np.float64).reshape(shape)),
                                   dtype=torch.float32).to(dev)

        g.positions = t(pos, (n, 3))
        g.rotations = t(rotations, (n, 4))
        g.log_scales = t(log_scales, (n, 3))
        g.opacity_logits = t(opacity_logits, (n,))
        g.sh_dc = t(sh[:, 0, :], (n, 3))
        g.sh_rest = t(sh[:, 1:, :], (n, 45))
        g.grad2d_accum = torch.zeros(n, dtype=torch.float32, device=dev)
        g.grad3d_accum = torch.zeros((n, 3), dtype=torch.float32, device=dev)
        g.obs_count = torch.zeros(n, dtype=torch.int32, device=dev)
        if not bool(torch.isfinite(g.sh_rest).all()):
            # sh_rest is validated here once; the preprocess kernel re-checks
            # it every forward only when it is optimised (sh_degree > 0)
            bad = int(torch.nonzero(~torch.isfinite(g.sh_rest).all(1))[0, 0])
            raise ValueError(f"non-finite parameter in primitive {bad}")
        return g

    @classmethod
    def from_scene(cls, sc, device=None) -> "GaussianMap":
        return cls.from_arrays(sc.positions, sc.rotations, sc.log_scales, sc.opacity_logits,
                               sc.sh, device)

    @property
    def sh(self) -> torch.Tensor:
        """(N, 16, 3) view assembled from sh_dc / sh_rest (a copy)."""
        n = len(self)
        return torch.cat([self.sh_dc.view(n, 1, 3), self.sh_rest.view(n, 15, 3)], dim=1)

    def opacities(self) -> torch.Tensor:
        return torch.sigmoid(self.opacity_logits)

    def scales(self) -> torch.Tensor:
        return torch.exp(self.log_scales)

    def to_numpy(self) -> dict:
        """Float64 host copy with the reference's array names."""
        return dict(positions=self.positions.double().cpu().numpy(),
                    rotations=self.rotations.double().cpu().numpy(),
                    log_scales=self.log_scales.double().cpu().numpy(),
                    opacity_logits=self.opacity_logits.double().cpu().numpy(),
                    sh=self.sh.double().cpu().numpy(),
                    grad2d_accum=self.grad2d_accum.double().cpu().numpy(),
                    grad3d_accum=self.grad3d_accum.double().cpu().numpy(),
                    obs_count=self.obs_count.long().cpu().numpy())

    def first_nonfinite_index(self):
        """core.py:231-241."""
        ok = (torch.isfinite(self.positions).all(1) & torch.isfinite(self.rotations).all(1)
              & torch.isfinite(self.log_scales).all(1) & torch.isfinite(self.opacity_logits)
              & torch.isfinite(self.sh_dc).all(1) & torch.isfinite(self.sh_rest).all(1))
        bad = torch.nonzero(~ok)
        return int(bad[0, 0]) if bad.numel() else None

    def normalize_rotations(self):
        """core.py:225-229."""
        nrm = torch.linalg.norm(self.rotations, dim=1, keepdim=True)
        if bool((nrm == 0).any()):
            raise ValueError("zero-norm quaternion in map")
        self.rotations /= nrm

    def reset_grad_stats(self):
        """core.py:219-223."""
        self.grad2d_accum.zero_()
        self.grad3d_accum.zero_()
        self.obs_count.zero_()

    def keep_mask(self, keep) -> "GaussianMap":
        """core.py:200-209."""
        keep = torch.as_tensor(keep, device=self.device, dtype=torch.bool)
        for f in self.FIELDS:
            setattr(self, f, getattr(self, f)[keep].contiguous())
        return self

    def insert_arrays(self, positions, rotations, log_scales, opacity_logits, sh):
        """core.py:168-185 (new primitives start with zeroed statistics)."""
        other = GaussianMap.from_arrays(positions, rotations, log_scales, opacity_logits, sh,
                                        self.device)
        for f in self.FIELDS:
            setattr(self, f, torch.cat([getattr(self, f), getattr(other, f)]).contiguous())
        return self

    def insert_device(self, positions, rotations, log_scales, opacity_logits, sh_dc,
                      sh_rest=None):
        """insert_arrays for float32 device tensors (no host round trip);
        sh_rest defaults to zeros (seeded primitives, densify.py:79-81)."""
        n = int(positions.shape[0])
        if sh_rest is None:
            sh_rest = torch.zeros((n, 45), dtype=torch.float32, device=self.device)
        new = dict(positions=positions.reshape(n, 3), rotations=rotations.reshape(n, 4),
                   log_scales=log_scales.reshape(n, 3), opacity_logits=opacity_logits.reshape(n),
                   sh_dc=sh_dc.reshape(n, 3), sh_rest=sh_rest.reshape(n, 45),
                   grad2d_accum=torch.zeros(n, dtype=torch.float32, device=self.device),
                   grad3d_accum=torch.zeros((n, 3), dtype=torch.float32, device=self.device),
                   obs_count=torch.zeros(n, dtype=torch.int32, device=self.device))
        for f in self.FIELDS:
            setattr(self, f, torch.cat([getattr(self, f), new[f]]).contiguous())
        return self

    def ss(self) -> _lib.SSMap:
        m = _lib.SSMap()
        m.n = len(self)
        for f, name in (("positions", "d_positions"), ("rotations", "d_rotations"),
                        ("log_scales", "d_log_scales"), ("opacity_logits", "d_opacity_logits"),
                        ("sh_dc", "d_sh_dc"), ("sh_rest", "d_sh_rest"),
                        ("grad2d_accum", "d_grad2d_accum"), ("grad3d_accum", "d_grad3d_accum"),
                        ("obs_count", "d_obs_count")):
            t = getattr(self, f)
            assert t.is_contiguous() and t.is_cuda
            setattr(m, name, t.data_ptr() if t.numel() else None)
        return m

    def clone(self) -> "GaussianMap":
        g = GaussianMap(0, self.device)
        for f in self.FIELDS:
            setattr(g, f, getattr(self, f).clone())
        return g
