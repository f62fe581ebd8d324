"""Shared test helpers: golden fixture loading and parity metrics."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Cam:
    """Duck-typed camera accepted by the oracle and the product API."""

    def __init__(self, fx, fy, cx, cy, width, height, R, t):
        self.fx, self.fy, self.cx, self.cy = float(fx), float(fy), float(cx), float(cy)
        self.width, self.height = int(width), int(height)
        self.R = np.asarray(R, np.float64).reshape(3, 3)
        self.t = np.asarray(t, np.float64).reshape(3)

    @property
    def center(self):
        return -self.R.T @ self.t


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def fixture_camera(d):
    return Cam(d["cam_fx"], d["cam_fy"], d["cam_cx"], d["cam_cy"], int(d["width"]),
               int(d["height"]), d["cam_R"], d["cam_t"])


def fixture_scene(d):
    """Inputs of an iteration fixture (stored, or regenerated + checksummed)."""
    from paper_2410_00486_b200.scene import survey_scene

    if "in_positions" in d:
        return (d["in_positions"], d["in_rotations"], d["in_log_scales"],
                d["in_opacity_logits"], d["in_sh"])
    sc = survey_scene(int(d["n"]), int(d["seed"]))
    chk = np.array([sc.positions.sum(), sc.rotations.sum(), sc.log_scales.sum(),
                    sc.opacity_logits.sum(), sc.sh.sum()])
    np.testing.assert_allclose(chk, d["in_checksum"], rtol=0, atol=1e-9)
    return sc.positions, sc.rotations, sc.log_scales, sc.opacity_logits, sc.sh


def expand_sh(a):
    """Fixtures store SH0 arrays with only the DC band."""
    if a.shape[1] == 16:
        return a
    out = np.zeros((a.shape[0], 16, 3))
    out[:, :a.shape[1]] = a
    return out


def normwise(a, b):
    """||a - b|| / ||b|| (the gradient metric)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def floored_rel(a, b, floor_frac=1e-3):
    """Largest elementwise relative error over entries with |b| above
    floor_frac * max|b|."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if b.size == 0:
        return 0.0
    mx = np.abs(b).max()
    if mx == 0:
        return float(np.abs(a).max())
    sel = np.abs(b) > floor_frac * mx
    if not sel.any():
        return 0.0
    return float((np.abs(a[sel] - b[sel]) / np.abs(b[sel])).max())
