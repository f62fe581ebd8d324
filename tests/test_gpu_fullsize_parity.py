"""Stage-wise parity against the CPU oracle at the BASELINE.json sizes
(SURVEY.md 8c protocol, north_star tolerances):

=============  ============================================  ==========
config         scene                                          SH
=============  ============================================  ==========
replica        S(300k), 1200x680  (configs[1], the headline)  0
tum            S(150k), 640x480   (configs[2])                0
large          S(1M),   1200x680  (configs[3], one view)      0
sh3            S(500k), 1200x680  (configs[4])                3
=============  ============================================  ==========

Each stage is fed the GPU's own float32 upstream values (a
float64 projection reorders thousands of depth ties, so the list must be
the GPU's), and compared with the oracle (oracle/, float64) stage by stage:

* K1 preprocess (projection.py:73-163): visible set equal; mean2d <= 1e-3
  px; cov2d / conic <= 1e-5 of the column max; depth, sigma, rgb <= 1e-5;
  radius flips counted (float32 rounding at the ceil boundary);
* K2-K4b binning (tiles.py:29-65): pair list, tile ranges and active tiles
  BIT-EXACT;
* K5 blend (kernels.py:34-109): image and final_T <= 1e-4 absolute at
  every pixel clear of the blend's discrete decisions (the oracle flags
  pixels with an evaluation within BAND of m_cut / alpha_min / t_min);
  n_contrib flips only at flagged pixels, k_eff equal outside their tiles;
* K6 loss (losses.py:198-228): scalars <= 1e-6 rel, grad_image <= 1e-5
  norm-wise and max-abs;
* K7 splat-wise backward (kernels.py:271-373) and K8 chain
  (projection.py:200-325): <= 1e-3 norm-wise AND <= 1e-3 elementwise on
  entries above 1e-3 x max (for K7 over the rows not blended at
  a flagged threshold pixel);
* K9 Adam (optimizer.py:101-133), all six groups incl. the quaternion
  renorm and sh_rest, from non-zero moments: each parameter's step within
  1e-3 of the oracle's step (plus two float32 ulps of the parameter, four
  for the renormalised quaternions);
* fused K8+K9 (the engine's chain_adam kernel) over one engine step vs the
  oracle chain + regulariser + Adam on the engine's own g2d;
* K10 densify (densify.py:103-173): survivors, counts bit-exact.

Set SS_PARITY_REPORT=<path> to append every measured figure as a JSON line
(profiles/r02_parity_fullsize.jsonl was made that way).
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle as orc  # noqa: E402
from helpers import floored_rel, normwise  # noqa: E402

# relative band around the blend's discrete decisions (m_cut, alpha_min,
# t_min) inside which float32 and float64 may decide differently; the GPU's
# alpha is within ~5e-7 relative of the exact value (ex2.approx), its
# quadratic form within ~1e-6
BAND = 5e-6

CONFIGS = {
    "replica": (300_000, 1200, 680, 0),
    "tum": (150_000, 640, 480, 0),
    "large": (1_000_000, 1200, 680, 0),
    "sh3": (500_000, 1200, 680, 3),
}


def report(cfg, stage, **kv):
    path = os.environ.get("SS_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(dict(config=cfg, stage=stage, **{
                k: (float(v) if isinstance(v, (np.floating, float)) else
                    int(v) if isinstance(v, (np.integer, int)) else v)
                for k, v in kv.items()})) + "\n")


def _f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


@pytest.fixture(scope="module", params=list(CONFIGS))
def fs(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    orc.set_threads(os.cpu_count() or 1)
    name = request.param
    n, w, h, deg = CONFIGS[name]
    cam = survey_camera(w, h)
    opts = ss.RasterOpts(sh_degree=deg)
    sc = survey_scene(n, 0)
    tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam,
                               opts).image.clone()
    g = ss.GaussianMap.from_scene(sc)
    out = ss.rasterize_forward(g, cam, opts)
    torch.cuda.synchronize()
    om = orc.OMap(_f32(sc.positions), _f32(sc.rotations), _f32(sc.log_scales),
                  _f32(sc.opacity_logits), _f32(sc.sh))
    ctx = dict(name=name, ss=ss, cam=cam, opts=opts, sc=sc, tgt=tgt, g=g, out=out, om=om,
               deg=deg, n=n)
    yield ctx
    ctx.clear()
    torch.cuda.empty_cache()


def _oracle_forward(fs):
    """orc.forward on the GPU's float32 projection and pair list."""
    if "r" not in fs:
        out, cam = fs["out"], fs["cam"]
        p = out.proj
        po = orc.OProjection(map_index=p.map_index, t_cam=p.t_cam.astype(np.float64),
                             depth=p.depth.astype(np.float64),
                             mean2d=p.mean2d.astype(np.float64),
                             cov2d=p.cov2d.astype(np.float64), conic=p.conic.astype(np.float64),
                             radius=p.radius.astype(np.float64), sigma=p.sigma.astype(np.float64),
                             rgb=p.rgb.astype(np.float64), rgb_active=p.rgb_active,
                             sh_degree=p.sh_degree)
        ti = out.tile_index
        oti = orc.OTileIndex(16, ti.tiles_x, ti.tiles_y, ti.pair_splat, ti.tile_range,
                             ti.active_tiles)
        fs["r"] = orc.forward(po, oti, cam.width, cam.height, out.n_primitives,
                              m_cut=p.m_cut.astype(np.float64), threshold_band=BAND)
    return fs["r"]


def _threshold_rows(fs):
    """Projection rows blended (by the GPU or the oracle) at a flagged
    threshold pixel: their g2d rows get that pixel's terms, which a float32
    threshold decision may legitimately change."""
    if "thr_rows" not in fs:
        out, r = fs["out"], _oracle_forward(fs)
        ti = out.tile_index
        nc = np.maximum(out.n_contrib.cpu().numpy(), r.n_contrib)
        rows = set()
        for y, x in zip(*np.nonzero(r.extra["threshold_px"])):
            tid = (y // 16) * ti.tiles_x + x // 16
            a = int(ti.tile_range[tid])
            rows.update(ti.pair_splat[a:a + int(nc[y, x])].tolist())
        fs["thr_rows"] = np.array(sorted(rows), dtype=np.int64)
    return fs["thr_rows"]


def _loss(fs):
    if "lb" not in fs:
        ss = fs["ss"]
        fs["lb"] = ss.compute_losses(fs["out"].image, fs["tgt"], fs["g"].opacity_logits,
                                     0.2, 0.001)
    return fs["lb"]


def _g2d(fs):
    """K7 on the real loss gradient of this render."""
    if "g2d" not in fs:
        fs["g2d"] = fs["ss"].screen_space_grads(fs["out"], _loss(fs).grad_image)
    return fs["g2d"]


def test_preprocess_vs_oracle(fs):
    out, cam, om, deg = fs["out"], fs["cam"], fs["om"], fs["deg"]
    ref = orc.project(om, cam, sh_degree=deg)
    fs["oproj"] = ref
    p = out.proj
    np.testing.assert_array_equal(p.map_index, ref.map_index)
    m2 = float(np.abs(p.mean2d - ref.mean2d).max())
    cov = max(float((np.abs(getattr(p, k) - getattr(ref, k))
                     / np.abs(getattr(ref, k)).max(axis=0)).max()) for k in ("conic", "cov2d"))
    dep = float((np.abs(p.depth - ref.depth) / np.abs(ref.depth)).max())
    sig = float((np.abs(p.sigma - ref.sigma) / np.abs(ref.sigma)).max())
    rgb = float(np.abs(p.rgb - ref.rgb).max())
    flips = int((p.radius != ref.radius).sum())
    report(fs["name"], "K1_preprocess", visible=len(ref), mean2d_abs=m2, cov_conic_rel=cov,
           depth_rel=dep, sigma_rel=sig, rgb_abs=rgb, radius_flips=flips)
    assert m2 <= 1e-3 and cov <= 1e-5 and dep <= 1e-5 and sig <= 1e-5 and rgb <= 1e-5
    # f32 vs f64 at the ceil(3 sigma) boundary (2 of 289,157 at 300k)
    assert flips <= max(4, len(ref) // 50_000)
    np.testing.assert_array_equal(p.rgb_active, ref.rgb_active)


def test_binning_bit_exact_vs_oracle(fs):
    out, cam = fs["out"], fs["cam"]
    p = out.proj
    ti = orc.tile_index(p.mean2d.astype(np.float32), p.radius.astype(np.float32),
                        p.depth.astype(np.float32), cam.width, cam.height, 16)
    g = out.tile_index
    report(fs["name"], "K2_K4b_binning", pairs=int(ti.pair_splat.size),
           active_tiles=int(ti.active_tiles.size),
           pair_mismatches=int((g.pair_splat != ti.pair_splat).sum())
           if g.pair_splat.size == ti.pair_splat.size else -1)
    assert out.pair_count == ti.pair_splat.size
    np.testing.assert_array_equal(g.pair_splat, ti.pair_splat)
    np.testing.assert_array_equal(g.tile_range, ti.tile_range)
    np.testing.assert_array_equal(g.active_tiles, ti.active_tiles)


def test_forward_vs_oracle(fs):
    """K5 on the GPU's list: colour / final_T within 1e-4 absolute at every
    pixel whose evaluations all lie clear of the blend's discrete decisions
    ("n_contrib equal except flagged threshold pixels"); the
    flagged pixels are counted, every n_contrib flip must be one of them,
    and there the difference is bounded by the few splats a flipped
    decision can add or drop (alpha_min = 1/255 each)."""
    out = fs["out"]
    r = _oracle_forward(fs)
    thr = r.extra["threshold_px"]
    img = out.image.cpu().numpy()
    ft = out.final_t.cpu().numpy()
    nc = out.n_contrib.cpu().numpy()
    d_img = np.abs(img - r.image).max(axis=2)
    d_t = np.abs(ft - r.final_t)
    e_img = float(d_img[~thr].max())
    e_t = float(d_t[~thr].max())
    e_img_thr = float(d_img[thr].max()) if thr.any() else 0.0
    flipped = nc != r.n_contrib
    flips = int(flipped.sum())
    ti = out.tile_index
    ke = out.k_eff
    H, W = nc.shape
    # tiles holding a flagged pixel may change k_eff; every other tile equal
    fl_tiles = set(((y // 16) * ti.tiles_x + x // 16) for y, x in zip(*np.nonzero(thr)))
    ok = np.array([t not in fl_tiles for t in ti.active_tiles])
    ke_mis = int((ke[ok] != r.k_eff[ok]).sum())
    contrib_mis = int((out.contributed.cpu().numpy() != r.contributed).sum())
    report(fs["name"], "K5_blend", image_abs=e_img, final_t_abs=e_t,
           image_abs_all_pixels=float(d_img.max()), threshold_pixels=int(thr.sum()),
           image_abs_threshold_pixels=e_img_thr, n_contrib_flips=flips,
           n_contrib_flips_unflagged=int((flipped & ~thr).sum()), pixels=H * W,
           k_eff_mismatch_outside_flagged_tiles=ke_mis, contributed_mismatch=contrib_mis)
    assert e_img <= 1e-4 and e_t <= 1e-4
    assert int((flipped & ~thr).sum()) == 0
    assert thr.sum() <= H * W // 1000
    assert e_img_thr <= 0.05
    assert ke_mis == 0
    assert contrib_mis <= 4 * flips + 2


def test_loss_vs_oracle(fs):
    lb = _loss(fs)
    out, tgt, g = fs["out"], fs["tgt"], fs["g"]
    ref = orc.losses(out.image.cpu().numpy().astype(np.float64),
                     tgt.cpu().numpy().astype(np.float64),
                     g.opacity_logits.cpu().numpy().astype(np.float64), 0.2, 0.001)
    rel = {k: abs(getattr(lb, k) - getattr(ref, k)) / max(abs(getattr(ref, k)), 1e-3)
           for k in ("l1", "ssim_loss", "rendered", "opacity_reg", "total")}
    gi = lb.grad_image.cpu().numpy()
    nw = normwise(gi, ref.grad_image)
    mx = float(np.abs(gi - ref.grad_image).max() / np.abs(ref.grad_image).max())
    report(fs["name"], "K6_loss", grad_normwise=nw, grad_maxabs_over_max=mx,
           **{f"{k}_rel": v for k, v in rel.items()})
    assert max(rel.values()) <= 1e-6, rel
    assert nw <= 1e-5 and mx <= 1e-5


def test_backward_g2d_vs_oracle(fs):
    """K7 on the real loss gradient; the oracle runs backward_splat on its
    own forward of the GPU's list (_oracle_forward)."""
    out = fs["out"]
    G = _loss(fs).grad_image
    mine = _g2d(fs).cpu().numpy().astype(np.float64)[out.proj.map_index]
    r = _oracle_forward(fs)
    ref = orc.backward_splat(r, G.cpu().numpy().astype(np.float64))
    fs["g2d_ref"] = ref
    # elementwise: rows not blended at a flagged threshold pixel (norm-wise: all rows)
    keep = np.ones(len(ref), bool)
    keep[_threshold_rows(fs)] = False
    res = {}
    for nm, cols in (("rgb", slice(0, 3)), ("mean2d", slice(3, 5)), ("conic", slice(5, 8)),
                     ("sigma", slice(8, 9))):
        res[nm] = (normwise(mine[:, cols], ref[:, cols]),
                   floored_rel(mine[keep, cols], ref[keep, cols], 1e-3))
    report(fs["name"], "K7_backward_g2d", **{f"{k}_normwise": v[0] for k, v in res.items()},
           **{f"{k}_elementwise_above_floor": v[1] for k, v in res.items()},
           rows=len(ref), rows_at_threshold_pixels=int((~keep).sum()))
    for k, (nw, el) in res.items():
        assert nw <= 1e-3, (k, nw)
        assert el <= 1e-3, (k, el)


def test_chain_vs_oracle(fs):
    """K8 on the GPU's own g2d (chain_backward, projection.py:200-299)."""
    ss, out, cam, om, deg = fs["ss"], fs["out"], fs["cam"], fs["om"], fs["deg"]
    g2d = _g2d(fs)
    grads = ss.rasterizer._finish_backward(out, g2d)
    fs["grads"] = grads
    po = fs.get("oproj") or orc.project(om, cam, sh_degree=deg)
    ref = orc.chain(om, cam, po, g2d.cpu().numpy().astype(np.float64)[out.proj.map_index],
                    out.contributed.cpu().numpy())
    res = {}
    for name in ("position", "rotation", "log_scale", "opacity_logit", "pos2d_grad_norm"):
        a = getattr(grads, name).cpu().numpy()
        b = getattr(ref, name)
        res[name] = (normwise(a, b), floored_rel(a, b, 1e-3))
    sh = grads.sh.cpu().numpy()
    res["sh_dc"] = (normwise(sh[:, 0], ref.sh[:, 0]), floored_rel(sh[:, 0], ref.sh[:, 0], 1e-3))
    if deg:
        res["sh_rest"] = (normwise(sh[:, 1:], ref.sh[:, 1:]),
                          floored_rel(sh[:, 1:], ref.sh[:, 1:], 1e-3))
    report(fs["name"], "K8_chain", **{f"{k}_normwise": v[0] for k, v in res.items()},
           **{f"{k}_elementwise_above_floor": v[1] for k, v in res.items()})
    for k, (nw, el) in res.items():
        assert nw <= 1e-3, (k, nw)
        assert el <= 1e-3, (k, el)


def _ulp(a):
    return np.spacing(np.abs(np.asarray(a, np.float32))).astype(np.float64)


def test_adam_all_groups_vs_oracle(fs):
    """adam_step from non-zero moments at step 7 on identical float32
    gradients (the chain's), every group incl. rotations + renorm and
    sh_rest: each parameter's step equals the oracle's within 1e-3 of the
    step plus 2 float32 ulps of the parameter; moments within 1e-5."""
    ss, om, deg, n = fs["ss"], fs["om"], fs["deg"], fs["n"]
    grads = fs.get("grads")
    if grads is None:
        grads = ss.rasterizer._finish_backward(fs["out"], _g2d(fs))
    if deg:
        # a non-trivial sh_rest gradient on every row (the chain's is only
        # non-zero for visible Gaussians)
        gen = torch.Generator(device="cuda").manual_seed(5)
        grads.sh_rest.add_(torch.randn(grads.sh_rest.shape, device="cuda", generator=gen) * 1e-5)
    g = ss.GaussianMap.from_scene(fs["sc"])
    st = ss.AdamState.for_map(g)
    rng = np.random.default_rng(9)
    ost = orc.OAdam.for_map(om)
    shapes = {"position": (n, 3), "rotation": (n, 4), "log_scale": (n, 3),
              "opacity_logit": (n,), "sh_dc": (n, 3), "sh_rest": (n, 45)}
    for k, shp in shapes.items():
        m = (rng.standard_normal(shp) * 1e-3).astype(np.float32)
        v = (rng.uniform(1e-8, 1e-5, shp)).astype(np.float32)
        if k == "sh_rest" and not deg:  # unused at SH0: g = m = v = 0
            m[:] = 0.0
            v[:] = 0.0
        st.m[k].copy_(torch.as_tensor(m).view(st.m[k].shape))
        st.v[k].copy_(torch.as_tensor(v).view(st.v[k].shape))
        ok = {"sh_dc": (n, 1, 3), "sh_rest": (n, 15, 3)}.get(k, ost.m[k].shape)
        ost.m[k] = m.astype(np.float64).reshape(ok)
        ost.v[k] = v.astype(np.float64).reshape(ok)
    st.step_count = ost.step_count = 6
    if deg:
        st.sh_rest_active = True
    pre = {f: getattr(g, f).cpu().numpy().astype(np.float64)
           for f in ("positions", "rotations", "log_scales", "opacity_logits", "sh_dc",
                     "sh_rest")}
    ss.adam_step(g, grads, st)
    og = orc.OGrads(*[getattr(grads, k).cpu().numpy().astype(np.float64) for k in
                      ("position", "rotation", "log_scale", "opacity_logit")],
                    grads.sh.cpu().numpy().astype(np.float64),
                    grads.pos2d_grad_norm.cpu().numpy().astype(np.float64),
                    grads.contributed.cpu().numpy())
    oref = om.copy()
    orc.adam(oref, og, ost)
    refs = {"positions": oref.positions, "rotations": oref.rotations,
            "log_scales": oref.log_scales, "opacity_logits": oref.opacity_logits,
            "sh_dc": oref.sh[:, 0, :], "sh_rest": oref.sh[:, 1:, :].reshape(n, 45)}
    res = {}
    for f, b in refs.items():
        a = getattr(g, f).cpu().numpy().astype(np.float64).reshape(b.shape)
        step_ref = b - pre[f].reshape(b.shape)
        err = np.abs(a - b)
        # the quaternion renorm adds 3 roundings (sum of squares, rsqrt, scale)
        bound = 1e-3 * np.abs(step_ref) + (4 if f == "rotations" else 2) * _ulp(b)
        res[f] = (float((err / np.maximum(bound, 1e-30)).max()),
                  float(np.abs(step_ref).max()))
    for k in shapes:
        a = st.m[k].cpu().numpy().reshape(-1)
        b = ost.m[k].reshape(-1)
        res[f"m_{k}"] = (float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30) / 1e-5), 0.0)
        a = st.v[k].cpu().numpy().reshape(-1)
        b = ost.v[k].reshape(-1)
        res[f"v_{k}"] = (float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30) / 1e-5), 0.0)
    report(fs["name"], "K9_adam", **{f"{k}_err_over_bound": v[0] for k, v in res.items()},
           **{f"{k}_max_step": v[1] for k, v in res.items() if v[1]})
    for k, (r, _) in res.items():
        assert r <= 1.0, (k, r)


def test_engine_fused_step_vs_oracle(fs):
    """One MappingEngine step (fused K8+K9 kernel, chain + regulariser +
    stats + Adam) vs the oracle's chain + adam + accumulate_grad_stats on the
    engine's own screen-space rows: first Adam step, so the step is
    lr * g / (|g| + eps): compared elementwise where |g_ref| is above
    1e-3 x max (float32 noise flips the sign of near-zero gradients)."""
    ss, cam, om, deg, n = fs["ss"], fs["cam"], fs["om"], fs["deg"], fs["n"]
    g = ss.GaussianMap.from_scene(fs["sc"])
    eng = ss.MappingEngine(g, cam.width, cam.height, fs["opts"])
    eng.fit_capacity(cam)
    eng.step(cam, fs["tgt"])
    eng.synchronize()
    g2d = eng.g2d.cpu().numpy().astype(np.float64)
    contrib = eng.contributed.cpu().numpy().astype(bool)
    po = fs.get("oproj") or orc.project(om, cam, sh_degree=deg)
    ref = orc.chain(om, cam, po, g2d[po.map_index], contrib)
    lref = orc.losses(fs["out"].image.cpu().numpy().astype(np.float64),
                      fs["tgt"].cpu().numpy().astype(np.float64), om.opacity_logits, 0.2, 0.001)
    ref.opacity_logit = ref.opacity_logit + lref.grad_opacity_logit
    oref = om.copy()
    orc.adam(oref, ref, orc.OAdam.for_map(oref))
    orc.accumulate_grad_stats(oref, ref)
    res = {}
    for f, gname, lr in (("positions", "position", 1.6e-4), ("rotations", "rotation", None),
                         ("log_scales", "log_scale", 5e-3),
                         ("opacity_logits", "opacity_logit", 5e-2)):
        a = getattr(g, f).cpu().numpy().astype(np.float64)
        b = getattr(oref, f)
        gr = getattr(ref, gname)
        sel = np.abs(gr) > 1e-3 * np.abs(gr).max()
        if f == "rotations":  # renormalised: compare the whole row where any entry is big
            sel = np.repeat(sel.any(axis=1, keepdims=True), 4, axis=1)
        pre = getattr(om, f)
        step_ref = b - pre
        err = np.abs(a - b)[sel]
        bound = 1e-3 * np.abs(step_ref)[sel] + (4 if f == "rotations" else 2) * _ulp(b)[sel]
        res[f] = float((err / bound).max()) if sel.any() else 0.0
        if lr is not None:  # every selected element moved by ~lr in the oracle's direction
            assert np.all(np.sign(a - pre)[sel] == np.sign(step_ref)[sel]), f
    nw_g2d = normwise(g.grad2d_accum.cpu().numpy(), oref.grad2d_accum)
    obs_ok = bool(np.array_equal(g.obs_count.cpu().numpy(), oref.obs_count))
    report(fs["name"], "K8K9_fused_engine_step",
           **{f"{k}_err_over_bound": v for k, v in res.items()},
           grad2d_accum_normwise=nw_g2d, obs_count_equal=obs_ok)
    for k, r in res.items():
        assert r <= 1.0, (k, r)
    assert nw_g2d <= 1e-3 and obs_ok
    fs["after_step"] = (g, eng)


def test_densify_bit_exact_vs_oracle(fs):
    """densify_and_prune at full size on the post-step map and statistics
    (float64 mask math on the stored float32 values): the
    survivors, clone/split/prune counts bit-exact; new rows to float32."""
    ss = fs["ss"]
    if "after_step" not in fs:
        pytest.skip("needs the engine step of test_engine_fused_step_vs_oracle")
    g, _ = fs["after_step"]
    h = g.to_numpy()
    om = orc.OMap(h["positions"], h["rotations"], h["log_scales"], h["opacity_logits"], h["sh"],
                  h["grad2d_accum"], h["grad3d_accum"], h["obs_count"])
    # thresholds at quantiles of this map so that all three masks are busy,
    # placed midway between two neighbouring data values (a threshold EQUAL
    # to a stored value would test the last ulp of exp(), which differs
    # between CUDA's and glibc's double exp; the reference's thresholds are
    # constants, not data values)
    def between(v, q):
        u = np.unique(v)
        k = int(q * (len(u) - 1))
        while k + 1 < len(u) and u[k + 1] - u[k] < 1e-9 * abs(u[k]):
            k += 1
        return float(0.5 * (u[k] + u[k + 1]))

    mean = om.grad2d_accum / np.maximum(om.obs_count, 1)
    thr = between(mean[om.obs_count > 0], 0.95)
    cfg = ss.DensifyConfig(grad_threshold=thr, prune_opacity=between(
        1 / (1 + np.exp(-om.opacity_logits)), 0.02))
    ext = between(np.exp(om.log_scales).max(axis=1), 0.5) / cfg.split_scale_percentile
    small, large, keep = orc.densify_masks(om, cfg.grad_threshold, cfg.prune_opacity,
                                           cfg.split_scale_percentile, ext)
    normals = np.random.default_rng(7).standard_normal((2 * int(large.sum()), 3))
    onew, ores = orc.densify_and_prune(om, normals=normals, grad_threshold=cfg.grad_threshold,
                                       prune_opacity=cfg.prune_opacity, scene_extent=ext)
    res = ss.densify_and_prune(g, cfg, ext, normals=normals)
    report(fs["name"], "K10_densify", n_in=len(om), n_out=len(onew), n_cloned=ores["n_cloned"],
           n_split=ores["n_split"], n_pruned=ores["n_pruned"],
           survivors_equal=bool(np.array_equal(res.survivors.cpu().numpy(),
                                               ores["survivors"])))
    assert ores["n_cloned"] > 0 and ores["n_split"] > 0 and ores["n_pruned"] > 0
    np.testing.assert_array_equal(res.survivors.cpu().numpy(), ores["survivors"])
    assert (res.n_new, res.n_cloned, res.n_split, res.n_pruned) == (
        ores["n_new"], ores["n_cloned"], ores["n_split"], ores["n_pruned"])
    hn = g.to_numpy()
    assert len(g) == len(onew)
    np.testing.assert_allclose(hn["positions"], onew.positions, rtol=0, atol=1e-5)
    np.testing.assert_allclose(hn["log_scales"], onew.log_scales, rtol=0, atol=1e-5)
    np.testing.assert_array_equal(hn["opacity_logits"].astype(np.float32),
                                  onew.opacity_logits.astype(np.float32))
