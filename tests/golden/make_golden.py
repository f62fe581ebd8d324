"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is read-only at /root/reference
and does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Every fixture is the output of the reference package `splatstream` itself
(float64, one worker, i.e. its deterministic mode), captured stage by stage
along one `_Trainer.train_one` iteration (trainer.py:180-215):
project_map -> build_tile_index -> rasterize_forward -> compute_losses ->
backward_splatwise (g2d captured by wrapping api._finish_backward) ->
+grad_opacity_logit -> adam_step -> accumulate_grad_stats, plus
backward_pixelwise, densify_and_prune/resize_for_densify and the SPEC.md
known-answer examples.  tests/test_oracle_golden.py pins oracle/ against
these files; the GPU tests then compare the CUDA path with the oracle.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = os.environ.get("SPLATSTREAM_REF", "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import splatstream as ss  # noqa: E402  (the reference)
from splatstream import densify as ref_densify  # noqa: E402
from splatstream import losses as ref_losses  # noqa: E402
from splatstream import optimizer as ref_opt  # noqa: E402
from splatstream.rasterizer import api as ref_api  # noqa: E402
from splatstream.rasterizer import projection as ref_proj  # noqa: E402
from splatstream.rasterizer import tiles as ref_tiles  # noqa: E402

from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402


def ref_map(sc):
    return ss.GaussianMap.from_arrays(sc.positions, sc.rotations, sc.log_scales,
                                      sc.opacity_logits, sc.sh)


def ref_cam(pc):
    return ss.Camera(pc.fx, pc.fy, pc.cx, pc.cy, pc.width, pc.height, R=pc.R, t=pc.t)


def capture_iteration(name, n, width, height, sh_degree, seed, view=0, n_views=1,
                      store_inputs=True, store_ckpt=True):
    sc = survey_scene(n, seed)
    tsc = survey_scene(n, seed + 100)
    pc = survey_camera(width, height, view, n_views)
    cam = ref_cam(pc)
    gmap = ref_map(sc)
    target = ss.rasterize_forward(ref_map(tsc), cam, ss.RasterOpts(
        sh_degree=sh_degree, with_checkpoints=False)).image
    opts = ss.RasterOpts(sh_degree=sh_degree)
    proj = ref_proj.project_map(gmap, cam, sh_degree=sh_degree)
    ti = ref_tiles.build_tile_index(proj, width, height, 16)
    out = ss.rasterize_forward(gmap, cam, opts)
    lb = ss.compute_losses(out.image, target, gmap.opacity_logits, 0.2, 0.001)
    cap = {}
    orig = ref_api._finish_backward

    def capture(render, g2d):
        cap["g2d"] = g2d.copy()
        return orig(render, g2d)

    ref_api._finish_backward = capture
    try:
        grads = ss.backward_splatwise(out, lb.grad_image)
    finally:
        ref_api._finish_backward = orig
    gpix = ss.backward_pixelwise(out, lb.grad_image)
    grads.opacity_logit = grads.opacity_logit + lb.grad_opacity_logit
    st = ref_opt.AdamState.for_map(gmap)
    ss.adam_step(gmap, grads, st)
    ref_densify.accumulate_grad_stats(gmap, grads)

    d = dict(
        width=width, height=height, sh_degree=sh_degree, seed=seed, view=view,
        n_views=n_views, n=n,
        cam_fx=pc.fx, cam_fy=pc.fy, cam_cx=pc.cx, cam_cy=pc.cy, cam_R=pc.R, cam_t=pc.t,
        in_checksum=np.array([sc.positions.sum(), sc.rotations.sum(), sc.log_scales.sum(),
                              sc.opacity_logits.sum(), sc.sh.sum()]),
        target=target,
        proj_map_index=proj.map_index, proj_mean2d=proj.mean2d, proj_cov2d=proj.cov2d,
        proj_conic=proj.conic, proj_radius=proj.radius, proj_sigma=proj.sigma,
        proj_rgb=proj.rgb, proj_rgb_active=proj.rgb_active, proj_depth=proj.depth,
        ti_pair_splat=ti.pair_splat, ti_tile_range=ti.tile_range,
        ti_active=ti.active_tiles,
        image=out.image, acc_rgb=out.acc_rgb, final_t=out.final_t, n_contrib=out.n_contrib,
        k_eff=out.k_eff, contributed=out.contributed, m_cut=out.m_cut,
        loss=np.array([lb.l1, lb.ssim_loss, lb.rendered, lb.opacity_reg, lb.total]),
        grad_image=lb.grad_image, grad_opacity_logit=lb.grad_opacity_logit,
        g2d=cap["g2d"],
        g_position=grads.position, g_rotation=grads.rotation, g_log_scale=grads.log_scale,
        g_opacity_logit=grads.opacity_logit, g_sh=grads.sh,
        g_pos2d_grad_norm=grads.pos2d_grad_norm,
        gpix_position=gpix.position, gpix_sh=gpix.sh, gpix_opacity_logit=gpix.opacity_logit,
        post_positions=gmap.positions, post_rotations=gmap.rotations,
        post_log_scales=gmap.log_scales, post_opacity_logits=gmap.opacity_logits,
        post_sh=gmap.sh, post_grad2d_accum=gmap.grad2d_accum,
        post_grad3d_accum=gmap.grad3d_accum, post_obs_count=gmap.obs_count,
        adam_m_position=st.m["position"], adam_v_position=st.v["position"],
        adam_m_sh_dc=st.m["sh_dc"], adam_v_rotation=st.v["rotation"],
    )
    if store_ckpt and out.checkpoints is not None:
        nbs = np.array([c.shape[0] for c in out.checkpoints], dtype=np.int64)
        d["ckpt_nb"] = nbs
        d["ckpt_flat"] = (np.concatenate([c.reshape(-1) for c in out.checkpoints])
                          if len(out.checkpoints) else np.zeros(0))
    if not store_ckpt:
        # large fixture: keep the stage outputs, drop what the small ones cover
        for k in ("gpix_position", "gpix_sh", "gpix_opacity_logit", "adam_m_position",
                  "adam_v_position", "adam_m_sh_dc", "adam_v_rotation", "acc_rgb",
                  "post_grad3d_accum", "proj_cov2d"):
            d.pop(k)
    if store_inputs:
        d.update(in_positions=sc.positions, in_rotations=sc.rotations,
                 in_log_scales=sc.log_scales, in_opacity_logits=sc.opacity_logits, in_sh=sc.sh)
    if sh_degree == 0:
        # SH0 keeps only the DC band meaningful; drop the 15 zero bands to
        # keep the fixture small (tests re-expand)
        for k in ("g_sh", "gpix_sh", "post_sh"):
            if k in d:
                d[k] = d[k][:, :1, :]
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **d)
    print(f"{name}: N={n} M={len(proj)} P={ti.pair_splat.size} "
          f"A={ti.active_tiles.size} size={os.path.getsize(path) / 1e6:.2f} MB")


def capture_densify(name="densify"):
    """densify_and_prune + resize_for_densify on a map with synthetic stats."""
    sc = survey_scene(600, 3)
    gmap = ref_map(sc)
    rng = np.random.default_rng(11)
    n = len(gmap)
    low = rng.random(n) < 0.1
    gmap.opacity_logits[low] = np.log(0.01) - np.log1p(-0.01)
    gmap.obs_count = rng.integers(0, 6, n).astype(np.int64)
    gmap.grad2d_accum = rng.uniform(0.0, 0.004, n) * gmap.obs_count
    gmap.grad3d_accum = rng.standard_normal((n, 3)) * 0.01
    pre = dict(pre_positions=gmap.positions.copy(), pre_rotations=gmap.rotations.copy(),
               pre_log_scales=gmap.log_scales.copy(),
               pre_opacity_logits=gmap.opacity_logits.copy(), pre_sh=gmap.sh.copy(),
               pre_grad2d_accum=gmap.grad2d_accum.copy(),
               pre_grad3d_accum=gmap.grad3d_accum.copy(), pre_obs_count=gmap.obs_count.copy())
    cfg = ref_densify.DensifyConfig()
    extent = 3.0
    st = ref_opt.AdamState.for_map(gmap)
    for k in st.m:
        st.m[k] = rng.standard_normal(st.m[k].shape)
        st.v[k] = rng.random(st.v[k].shape)
    m_pre = {k: v.copy() for k, v in st.m.items()}
    seed = 7
    res = ref_densify.densify_and_prune(gmap, cfg, extent, np.random.default_rng(seed))
    normals = np.random.default_rng(seed).standard_normal((res.n_split * cfg.split_children, 3))
    ref_opt.resize_for_densify(st, res.survivors, res.n_new)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"), extent=extent, normals=normals,
        survivors=res.survivors, n_new=res.n_new, n_cloned=res.n_cloned, n_split=res.n_split,
        n_pruned=res.n_pruned,
        post_positions=gmap.positions, post_rotations=gmap.rotations,
        post_log_scales=gmap.log_scales, post_opacity_logits=gmap.opacity_logits,
        post_sh=gmap.sh, post_obs_count=gmap.obs_count,
        m_pre_position=m_pre["position"], m_post_position=st.m["position"],
        v_post_rotation=st.v["rotation"], **pre)
    print(f"{name}: cloned={res.n_cloned} split={res.n_split} pruned={res.n_pruned} "
          f"new={res.n_new}")


def known_answers():
    """SPEC.md examples evaluated by the reference."""
    ka = {}
    ka["cov_ln2_x"] = ss.build_covariance([1, 0, 0, 0], [np.log(2), 0, 0]).tolist()
    c, s = np.cos(np.pi / 4), np.sin(np.pi / 4)
    ka["cov_rotz90"] = ss.build_covariance([c, 0, 0, s], [np.log(2), 0, 0]).tolist()
    ka["sh_zero"] = ss.eval_sh(np.zeros(48), [0, 0, 1], 0).tolist()
    dc = np.zeros((16, 3))
    dc[0] = (1, 0, 0)
    ka["sh_dc"] = ss.eval_sh(dc, [0, 0, 1], 0).tolist()
    cam = ss.Camera(100.0, 100.0, 64.0, 64.0, 128, 128)
    prim = ss.GaussianPrimitive([0, 0, 10], [1, 0, 0, 0], [0, 0, 0], 0.0, np.zeros(48))
    p2 = ss.project_gaussian(prim, cam)
    ka["proj_mean2d"] = p2.mean2d.tolist()
    ka["proj_cov2d"] = p2.cov2d.tolist()
    prim_b = ss.GaussianPrimitive([0, 0, -1], [1, 0, 0, 0], [0, 0, 0], 0.0, np.zeros(48))
    ka["proj_behind_culled"] = ss.project_gaussian(prim_b, cam) is None
    # empty map
    out = ss.rasterize_forward(ss.GaussianMap(), ss.Camera(50.0, 50.0, 16.0, 12.0, 32, 24))
    ka["empty_image_max"] = float(out.image.max())
    ka["empty_final_t_min"] = float(out.final_t.min())
    # loss arithmetic
    ka["opacity_reg"] = ss.opacity_reg(np.array([0.5, 0.25, 0.0, 1.0]))[0]
    ka["total_loss"] = ss.total_loss(0.18, 0.4375, 0.001)
    a0 = np.zeros((16, 16, 3))
    a1 = np.ones((16, 16, 3))
    ka["ssim_const_0_1"] = ss.ssim_metric(a0, a1)
    ka["psnr_same"] = ss.psnr(a0, a0)
    ka["psnr_mse_0.01"] = ss.psnr(a0, np.full_like(a0, 0.1))
    rl, _ = ss.rendered_loss(a1 * 0.5, a1 * 0.5)
    ka["rendered_loss_identical"] = rl
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(ka, f, indent=1, sort_keys=True)
    print("known answers:", len(ka))


def capture_loss_odd():
    """compute_losses on an image narrower than the SSIM window (exercises
    the repeated-reflection path, losses.py:31-41,58-66)."""
    rng = np.random.default_rng(5)
    x = rng.random((9, 14, 3))
    y = rng.random((9, 14, 3))
    lg = rng.standard_normal(17)
    lb = ss.compute_losses(x, y, lg, 0.2, 0.001)
    np.savez_compressed(os.path.join(HERE, "loss_small.npz"), x=x, y=y, logits=lg,
                        loss=np.array([lb.l1, lb.ssim_loss, lb.rendered, lb.opacity_reg,
                                       lb.total]),
                        grad_image=lb.grad_image, grad_opacity_logit=lb.grad_opacity_logit)
    print("loss_small done")


def capture_scheduler_and_metrics():
    """KeyframeScheduler traces (scheduler.py:22-89) and the eval metrics
    psnr / ssim_metric (losses.py:112-116,176-182) evaluated by the reference."""
    from splatstream.scheduler import KeyframeScheduler

    def loss_of(kf, step):
        return 1.0 / (1.0 + kf) + 0.01 * ((step * 7919) % 13)

    out = {}
    for d, r0, seed in ((4, 8, 0), (2, 3, 7)):
        sch = KeyframeScheduler(d=d, r0=r0, seed=seed)
        picks = []
        for step in range(240):
            if step % 10 == 0:
                sch.add_keyframe(step // 10)
            kf = sch.select()
            picks.append(int(kf))
            sch.record_result(kf, loss_of(kf, step))
        out[f"select_d{d}_r{r0}_s{seed}"] = picks
        out[f"remaining_d{d}_r{r0}_s{seed}"] = [int(r) for r in sch.remaining]
        base = KeyframeScheduler(d=d, r0=r0, seed=seed)
        for k in range(5):
            base.add_keyframe(k)
        out[f"uniform_d{d}_r{r0}_s{seed}"] = [int(base.select_uniform_baseline())
                                              for _ in range(50)]
    rng = np.random.default_rng(11)
    a = rng.random((20, 24, 3))
    b = np.clip(a + 0.05 * rng.standard_normal(a.shape), 0, 1)
    out["metrics_a"] = a.tolist()
    out["metrics_b"] = b.tolist()
    out["psnr_ab"] = ss.psnr(a, b)
    out["ssim_metric_ab"] = ss.ssim_metric(a, b)
    with open(os.path.join(HERE, "scheduler_metrics.json"), "w") as f:
        json.dump(out, f)
    print("scheduler/metrics done")


def capture_seed():
    """seed_from_points (densify.py:53-83) by the reference on float32-exact
    clouds: uniform, clustered with duplicates, and the n = 1, 2, 3 cases."""
    rng = np.random.default_rng(21)
    clouds = {
        "uniform": rng.uniform(-1.0, 1.0, (3000, 3)),
        "clustered": np.concatenate([rng.normal(c, 0.02, (400, 3))
                                     for c in rng.uniform(-2, 2, (5, 3))]),
        "n1": rng.uniform(-1, 1, (1, 3)),
        "n2": rng.uniform(-1, 1, (2, 3)),
        "n3": rng.uniform(-1, 1, (3, 3)),
    }
    clouds["clustered"][:10] = clouds["clustered"][10:20]  # exact duplicates
    out = {}
    for name, p in clouds.items():
        p = p.astype(np.float32).astype(np.float64)
        c = rng.uniform(0, 1, p.shape).astype(np.float32).astype(np.float64)
        pos, rot, ls, op, sh = ref_densify.seed_from_points(p, c, scene_extent=2.5)
        out[f"{name}_points"] = p
        out[f"{name}_colors"] = c
        out[f"{name}_log_scales"] = ls
        out[f"{name}_opacity"] = op
        out[f"{name}_sh_dc"] = sh[:, 0, :]
        out[f"{name}_rotations"] = rot
    np.savez_compressed(os.path.join(HERE, "seed.npz"), **out)
    print("seed done")


def capture_ply():
    """save_map (dataio.py:279-305) by the reference, double and float32
    layouts, of a small float32-exact SH3 map."""
    from splatstream import dataio as ref_io
    rng = np.random.default_rng(31)
    n = 40
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    rot = rng.standard_normal((n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    g = ss.GaussianMap()
    g.insert_arrays(f32(rng.uniform(-1, 1, (n, 3))), f32(rot), f32(rng.normal(-3, 0.3, (n, 3))),
                    f32(rng.normal(0, 1, n)), f32(rng.normal(0, 0.2, (n, 16, 3))))
    ref_io.save_map(g, os.path.join(HERE, "map_f64.ply"))
    ref_io.save_map(g, os.path.join(HERE, "map_f32.ply"), float32=True)
    print("ply done")


if __name__ == "__main__":
    capture_iteration("iter_sh0_small", 800, 64, 48, 0, seed=0)
    capture_iteration("iter_sh3_small", 600, 48, 40, 3, seed=1, view=1, n_views=3)
    capture_iteration("iter_tiny_config", 10_000, 128, 96, 0, seed=0, store_inputs=False,
                      store_ckpt=False)
    capture_densify()
    capture_loss_odd()
    known_answers()
    capture_scheduler_and_metrics()
    capture_seed()
    capture_ply()
    _ = ref_losses
