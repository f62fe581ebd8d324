"""Synthetic scene recipe and the oracle on it (CPU)."""

import numpy as np

import oracle as orc
from paper_2410_00486_b200.scene import SH_C0, survey_camera, survey_scene


def test_recipe_reproduces_survey_tiny_counts():
    """tiny config S(10k,128x96) has M=9980, P=36003, A=48."""
    sc = survey_scene(10_000, 0)
    cam = survey_camera(128, 96)
    om = orc.OMap(sc.positions, sc.rotations, sc.log_scales, sc.opacity_logits, sc.sh)
    p = orc.project(om, cam, sh_degree=0)
    ti = orc.tile_index(p.mean2d, p.radius, p.depth, 128, 96)
    assert len(p) == 9980
    assert ti.pair_splat.size == 36003
    assert ti.active_tiles.size == 48


def test_recipe_distributions():
    sc = survey_scene(5000, 1)
    assert np.allclose(np.linalg.norm(sc.rotations, axis=1), 1.0)
    assert sc.positions.min() >= -0.4 and sc.positions.max() <= 0.4
    op = 1 / (1 + np.exp(-sc.opacity_logits))
    assert op.min() >= 0.55 and op.max() <= 0.97
    base = sc.sh[:, 0, :] * SH_C0 + 0.5
    assert base.min() >= 0.1 and base.max() <= 0.9


def test_orbit_cameras_look_at_origin():
    for v in range(4):
        c = survey_camera(64, 48, v, 4)
        ctr = c.center
        assert abs(np.linalg.norm(ctr[[0, 2]]) - 1.2) < 1e-12
        z = c.R @ np.zeros(3) + c.t
        assert z[2] > 0 and abs(z[0]) < 1e-12 and abs(z[1]) < 1e-12
