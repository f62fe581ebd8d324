"""Synthetic Replica/TUM-shaped scenes (SURVEY.md 8d recipe).

Datasets are not available offline, so every benchmark and parity case
draws its map from ``gen_synthetic``'s distributions
(``dataio.py:370-382`` in the reference) with the scale shrunk as the map
grows so the footprint density stays scene-like, and renders from the
orbit camera the reference's generator uses (``dataio.py:384-399``).

Draw order with ``numpy.random.default_rng(seed)``:

1. ``pos = uniform(-0.4, 0.4, (N, 3))``
2. ``rot = standard_normal((N, 4))``, row-normalised
3. ``log_scale = log(uniform(0.02, 0.07, (N, 1)) * k)`` repeated to 3
   columns, ``+ log(uniform(0.6, 1.6, (N, 3)))`` with ``k = (500/N)^(1/3)``
4. ``opacity = uniform(0.55, 0.97, N)`` -> logit
5. ``sh = standard_normal((N, 16, 3)) * 0.015``;
   ``sh[:, 0, :] = (uniform(0.1, 0.9, (N, 3)) - 0.5) / SH_C0``
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SH_C0 = 0.28209479177387814

# BASELINE.json configs
CONFIGS = {
    "tiny": dict(n=10_000, width=128, height=96, sh_degree=0),
    "replica": dict(n=300_000, width=1200, height=680, sh_degree=0),
    "tum": dict(n=150_000, width=640, height=480, sh_degree=0),
    "large": dict(n=1_000_000, width=1200, height=680, sh_degree=0),
    "sh3": dict(n=500_000, width=1200, height=680, sh_degree=3),
}


@dataclass
class SceneArrays:
    """Float64 host arrays in the reference's layout (core.py:120-128)."""

    positions: np.ndarray   # (N, 3)
    rotations: np.ndarray   # (N, 4) w, x, y, z
    log_scales: np.ndarray  # (N, 3)
    opacity_logits: np.ndarray  # (N,)
    sh: np.ndarray          # (N, 16, 3) coefficient-major

    def __len__(self):
        return self.positions.shape[0]


def survey_scene(n: int, seed: int = 0) -> SceneArrays:
    """S(N, seed) of SURVEY.md 8d."""
    rng = np.random.default_rng(seed)
    k = (500.0 / n) ** (1.0 / 3.0)
    pos = rng.uniform(-0.4, 0.4, (n, 3))
    rot = rng.standard_normal((n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    ls = np.log(rng.uniform(0.02, 0.07, (n, 1)) * k).repeat(3, axis=1)
    ls += np.log(rng.uniform(0.6, 1.6, (n, 3)))
    op = rng.uniform(0.55, 0.97, n)
    logits = np.log(op) - np.log1p(-op)
    sh = rng.standard_normal((n, 16, 3)) * 0.015
    sh[:, 0, :] = (rng.uniform(0.1, 0.9, (n, 3)) - 0.5) / SH_C0
    return SceneArrays(pos, rot, ls, logits, sh)


@dataclass
class PinholeCamera:
    """Host camera with the reference's fields (core.py:244-301)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray
    t: np.ndarray

    @property
    def center(self) -> np.ndarray:
        return -self.R.T @ self.t


def looking_at(fx, fy, cx, cy, width, height, eye, target=(0.0, 0.0, 0.0),
               up=(0.0, 1.0, 0.0)) -> PinholeCamera:
    """Camera at ``eye`` with +z toward ``target`` (x right, y down),
    Camera.looking_at (core.py:287-301)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    up = np.asarray(up, dtype=np.float64)
    right = np.cross(fwd, up)
    if np.linalg.norm(right) < 1e-12:
        up = np.array([0.0, 0.0, 1.0]) if abs(fwd[1]) > 0.9 else np.array([0.0, 1.0, 0.0])
        right = np.cross(fwd, up)
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    return PinholeCamera(float(fx), float(fy), float(cx), float(cy), int(width), int(height),
                         R, -R @ eye)


def survey_camera(width: int, height: int, view: int = 0, n_views: int = 1,
                  theta0: float = 0.3, radius: float = 1.2, height_y: float = 0.35):
    """fx = fy = W / (2 tan 30 deg), principal point at the centre, eye on the
    orbit theta_v = theta0 + 2 pi v / V at radius 1.2."""
    fx = width / (2.0 * np.tan(np.deg2rad(30.0)))
    th = theta0 + 2.0 * np.pi * view / max(n_views, 1)
    eye = (radius * np.sin(th), height_y, radius * np.cos(th))
    return looking_at(fx, fx, width / 2.0, height / 2.0, width, height, eye)
