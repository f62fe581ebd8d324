"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import json
import os

import numpy as np
import pytest

import oracle as orc
from helpers import GOLDEN, expand_sh, fixture_camera, fixture_scene, load

ITER_FIXTURES = ["iter_sh0_small", "iter_sh3_small", "iter_tiny_config"]
RTOL = 1e-9   # float64 restatement vs float64 reference (summation order only)


def close(a, b, rtol=RTOL, atol_frac=1e-12):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    scale = max(float(np.abs(b).max()) if b.size else 0.0, 1e-300)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=atol_frac * scale)


@pytest.fixture(scope="module", params=ITER_FIXTURES)
def run(request):
    d = load(request.param)
    cam = fixture_camera(d)
    pos, rot, ls, op, sh = fixture_scene(d)
    gmap = orc.OMap(pos, rot, ls, op, sh)
    deg = int(d["sh_degree"])
    st = orc.OAdam.for_map(gmap)
    lb, inter = orc.iteration(gmap, cam, d["target"], st, sh_degree=deg, keep=True)
    return d, cam, gmap, st, lb, inter


def test_projection(run):
    d, cam, gmap, st, lb, inter = run
    p = inter["render"].proj
    np.testing.assert_array_equal(p.map_index, d["proj_map_index"])
    close(p.mean2d, d["proj_mean2d"])
    close(p.conic, d["proj_conic"])
    close(p.sigma, d["proj_sigma"])
    close(p.rgb, d["proj_rgb"])
    close(p.depth, d["proj_depth"])
    np.testing.assert_array_equal(p.radius, d["proj_radius"])
    np.testing.assert_array_equal(p.rgb_active, d["proj_rgb_active"])
    if "proj_cov2d" in d:
        close(p.cov2d, d["proj_cov2d"])


def test_tile_index_bit_exact(run):
    d, cam, gmap, st, lb, inter = run
    ti = inter["render"].tile_index
    np.testing.assert_array_equal(ti.pair_splat, d["ti_pair_splat"])
    np.testing.assert_array_equal(ti.tile_range, d["ti_tile_range"])
    np.testing.assert_array_equal(ti.active_tiles, d["ti_active"])


def test_forward(run):
    d, cam, gmap, st, lb, inter = run
    r = inter["render"]
    close(r.image, d["image"])
    close(r.final_t, d["final_t"])
    if "acc_rgb" in d:
        close(r.acc_rgb, d["acc_rgb"])
    np.testing.assert_array_equal(r.n_contrib, d["n_contrib"])
    np.testing.assert_array_equal(r.k_eff, d["k_eff"])
    np.testing.assert_array_equal(r.contributed, d["contributed"])
    close(r.m_cut, d["m_cut"])
    if "ckpt_flat" in d:
        cks = r.checkpoints()
        np.testing.assert_array_equal([c.shape[0] for c in cks], d["ckpt_nb"])
        close(np.concatenate([c.reshape(-1) for c in cks]), d["ckpt_flat"])


def test_losses(run):
    d, cam, gmap, st, lb, inter = run
    close([lb.l1, lb.ssim_loss, lb.rendered, lb.opacity_reg, lb.total], d["loss"], rtol=1e-10)
    close(lb.grad_image, d["grad_image"], rtol=1e-7, atol_frac=1e-10)
    close(lb.grad_opacity_logit, d["grad_opacity_logit"])


def test_backward_g2d(run):
    d, cam, gmap, st, lb, inter = run
    close(inter["g2d"], d["g2d"], rtol=1e-6, atol_frac=1e-9)


def test_param_grads(run):
    d, cam, gmap, st, lb, inter = run
    g = inter["grads"]
    for name in ("position", "rotation", "log_scale", "opacity_logit", "pos2d_grad_norm"):
        close(getattr(g, name), d["g_" + name], rtol=1e-6, atol_frac=1e-9)
    close(g.sh, expand_sh(d["g_sh"]), rtol=1e-6, atol_frac=1e-9)


def test_pixelwise_equals_splatwise(run):
    """SPEC.md:143,150 / acceptance #2: both backward modes agree; also
    against the reference's own pixel-wise result."""
    d, cam, gmap, st, lb, inter = run
    r = inter["render"]
    g2d_pix = orc.backward_pixel(r, lb.grad_image)
    close(g2d_pix, inter["g2d"], rtol=1e-9, atol_frac=1e-12)
    if "gpix_position" in d:
        gp = orc.chain(orc.OMap(*fixture_scene(d)), cam, r.proj, g2d_pix, r.contributed)
        close(gp.position, d["gpix_position"], rtol=1e-6, atol_frac=1e-9)


def test_adam_and_stats(run):
    d, cam, gmap, st, lb, inter = run
    close(gmap.positions, d["post_positions"], rtol=1e-12)
    close(gmap.rotations, d["post_rotations"], rtol=1e-12)
    close(gmap.log_scales, d["post_log_scales"], rtol=1e-12)
    close(gmap.opacity_logits, d["post_opacity_logits"], rtol=1e-12)
    close(gmap.sh[:, :d["post_sh"].shape[1]], d["post_sh"], rtol=1e-12)
    close(gmap.grad2d_accum, d["post_grad2d_accum"], rtol=1e-6, atol_frac=1e-9)
    np.testing.assert_array_equal(gmap.obs_count, d["post_obs_count"])
    if "adam_m_position" in d:
        close(st.m["position"], d["adam_m_position"], rtol=1e-6, atol_frac=1e-9)
        close(st.v["rotation"], d["adam_v_rotation"], rtol=1e-6, atol_frac=1e-9)


def test_checkpoint_replay_reproduces_final_state():
    """replaying from any checkpoint reproduces the forward."""
    d = load("iter_sh0_small")
    cam = fixture_camera(d)
    gmap = orc.OMap(*fixture_scene(d))
    r = orc.rasterize(gmap, cam, sh_degree=0)
    ti = r.tile_index
    for a in range(len(ti.active_tiles)):
        nb = (int(r.k_eff[a]) + 31) // 32
        x0, y0 = ti.tile_origin(ti.active_tiles[a])
        tw, th = min(16, r.width - x0), min(16, r.height - y0)
        for b in range(nb):
            T, rgb = orc.replay(r, a, b)
            np.testing.assert_array_equal(T, r.final_t[y0:y0 + th, x0:x0 + tw].reshape(-1))
            np.testing.assert_array_equal(rgb, r.acc_rgb[y0:y0 + th, x0:x0 + tw].reshape(-1, 3))


def test_bucket_partition_invariance():
    """SPEC.md:145 / acceptance #3: bucket size 32 vs 64 gives the same g2d."""
    d = load("iter_sh3_small")
    cam = fixture_camera(d)
    gmap = orc.OMap(*fixture_scene(d))
    r32 = orc.rasterize(gmap, cam, sh_degree=3, bucket=32)
    r64 = orc.rasterize(gmap, cam, sh_degree=3, bucket=64)
    g = np.random.default_rng(0).standard_normal(r32.image.shape)
    np.testing.assert_array_equal(orc.backward_splat(r32, g), orc.backward_splat(r64, g))


def test_thread_count_invariance():
    """api.py:1-7: results independent of the worker count."""
    d = load("iter_sh0_small")
    cam = fixture_camera(d)
    gmap = orc.OMap(*fixture_scene(d))
    g = np.random.default_rng(1).standard_normal((int(d["height"]), int(d["width"]), 3))
    old = orc.get_threads()
    outs = []
    for n in (1, 3):
        orc.set_threads(n)
        r = orc.rasterize(gmap, cam, sh_degree=0)
        outs.append((r.image, orc.backward_splat(r, g)))
    orc.set_threads(old)
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_loss_small_image_reflection():
    d = load("loss_small")
    lb = orc.losses(d["x"], d["y"], d["logits"], 0.2, 0.001)
    close([lb.l1, lb.ssim_loss, lb.rendered, lb.opacity_reg, lb.total], d["loss"], rtol=1e-10)
    close(lb.grad_image, d["grad_image"], rtol=1e-8, atol_frac=1e-12)
    close(lb.grad_opacity_logit, d["grad_opacity_logit"])


def test_densify_and_resize():
    d = load("densify")
    gmap = orc.OMap(d["pre_positions"], d["pre_rotations"], d["pre_log_scales"],
                    d["pre_opacity_logits"], d["pre_sh"], d["pre_grad2d_accum"].copy(),
                    d["pre_grad3d_accum"].copy(), d["pre_obs_count"].copy())
    new, res = orc.densify_and_prune(gmap, normals=d["normals"], scene_extent=float(d["extent"]))
    np.testing.assert_array_equal(res["survivors"], d["survivors"])
    assert res["n_new"] == int(d["n_new"])
    assert res["n_cloned"] == int(d["n_cloned"])
    assert res["n_split"] == int(d["n_split"])
    assert res["n_pruned"] == int(d["n_pruned"])
    close(new.positions, d["post_positions"], rtol=1e-12)
    close(new.rotations, d["post_rotations"], rtol=0)
    close(new.log_scales, d["post_log_scales"], rtol=0)
    close(new.opacity_logits, d["post_opacity_logits"], rtol=0)
    close(new.sh, d["post_sh"], rtol=0)
    st = orc.OAdam.for_map(gmap)
    st.m["position"] = d["m_pre_position"].copy()
    orc.resize_for_densify(st, res["survivors"], res["n_new"])
    np.testing.assert_array_equal(st.m["position"], d["m_post_position"])


def test_known_answers():
    with open(os.path.join(GOLDEN, "known_answers.json")) as f:
        ka = json.load(f)
    # projection of an on-axis splat
    cam = type("C", (), dict(fx=100.0, fy=100.0, cx=64.0, cy=64.0, width=128, height=128,
                             R=np.eye(3), t=np.zeros(3)))()
    g = orc.OMap(np.array([[0, 0, 10.0]]), np.array([[1.0, 0, 0, 0]]), np.zeros((1, 3)),
                 np.zeros(1), np.zeros((1, 16, 3)))
    p = orc.project(g, cam)
    np.testing.assert_allclose(p.mean2d[0], ka["proj_mean2d"], rtol=1e-15)
    a, b, c = p.cov2d[0]
    np.testing.assert_allclose([[a, b], [b, c]], ka["proj_cov2d"], rtol=1e-14)
    gb = orc.OMap(np.array([[0, 0, -1.0]]), np.array([[1.0, 0, 0, 0]]), np.zeros((1, 3)),
                  np.zeros(1), np.zeros((1, 16, 3)))
    assert (len(orc.project(gb, cam)) == 0) == ka["proj_behind_culled"]
    # empty map: black image, T = 1
    cam2 = type("C", (), dict(fx=50.0, fy=50.0, cx=16.0, cy=12.0, width=32, height=24,
                              R=np.eye(3), t=np.zeros(3)))()
    e = orc.OMap(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                 np.zeros((0, 16, 3)))
    r = orc.rasterize(e, cam2)
    assert r.image.max() == ka["empty_image_max"]
    assert r.final_t.min() == ka["empty_final_t_min"]
    # loss arithmetic
    lb = orc.losses(np.zeros((4, 4, 3)), np.zeros((4, 4, 3)),
                    np.log(np.array([0.5, 0.25, 1e-300, 1 - 1e-16])) * 0 + np.array(
                        [0.0, np.log(0.25 / 0.75), -800.0, 800.0]), 0.2, 0.001)
    assert abs(lb.opacity_reg - ka["opacity_reg"]) < 1e-12
    assert abs(ka["total_loss"] - (0.18 + 0.001 * 0.4375)) < 1e-15
    lb2 = orc.losses(np.full((6, 6, 3), 0.5), np.full((6, 6, 3), 0.5), np.zeros(1))
    assert lb2.rendered == ka["rendered_loss_identical"]


def test_two_splat_blend_known_answer():
    """(1,0,0)@0.5 then (0,1,0)@0.5 -> (0.5,0.25,0), T=0.25."""
    p = orc.OProjection(map_index=np.array([0, 1], np.int32), t_cam=np.zeros((2, 3)),
                        depth=np.array([1.0, 2.0]), mean2d=np.array([[0.0, 0.0], [0.0, 0.0]]),
                        cov2d=np.zeros((2, 3)), conic=np.zeros((2, 3)),
                        radius=np.array([1.0, 1.0]), sigma=np.array([0.5, 0.5]),
                        rgb=np.array([[1.0, 0, 0], [0, 1.0, 0]]),
                        rgb_active=np.ones((2, 3), bool))
    ti = orc.tile_index(p.mean2d, p.radius, p.depth, 4, 4)
    r = orc.forward(p, ti, 4, 4, 2)
    np.testing.assert_allclose(r.image[0, 0], [0.5, 0.25, 0.0])
    assert r.final_t[0, 0] == 0.25
    assert r.n_contrib[0, 0] == 2


@pytest.mark.parametrize("cloud", ["uniform", "clustered", "n1", "n2", "n3"])
def test_oracle_seed_from_points_matches_reference(cloud):
    """F3 seeding restatement vs the reference's seed_from_points outputs."""
    d = np.load(os.path.join(GOLDEN, "seed.npz"))
    pos, rot, ls, op, sh = orc.seed_from_points(d[f"{cloud}_points"], d[f"{cloud}_colors"],
                                                scene_extent=2.5)
    np.testing.assert_allclose(ls, d[f"{cloud}_log_scales"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(op, d[f"{cloud}_opacity"], rtol=1e-15)
    np.testing.assert_allclose(sh[:, 0, :], d[f"{cloud}_sh_dc"], rtol=1e-14)
    np.testing.assert_array_equal(rot, d[f"{cloud}_rotations"])
