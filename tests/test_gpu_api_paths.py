"""The drop-in API's own fast paths: contributed derived from the blend
masks, the one-launch finite check, and adam_step's reuse of
backward_splatwise's eager check (only tensors modified since are
re-checked)."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _scene(n=20000, w=320, h=240, seed=11):
    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    cam = survey_camera(w, h)
    g = ss.GaussianMap.from_scene(survey_scene(n, seed))
    return ss, g, cam


def test_contributed_from_masks_equals_blend_loop_flag():
    """RenderOutput.contributed (ss_contributed_from_masks) == the flag the
    blend loop sets per blended pair (ss_blend_forward with d_contributed),
    bit for bit (kernels.py:94-95)."""
    _need_gpu()
    from paper_2410_00486_b200 import _lib
    from paper_2410_00486_b200.rasterizer import P, stream_handle
    ss, g, cam = _scene()
    out = ss.rasterize_forward(g, cam, ss.RasterOpts(sh_degree=0))
    lazy = out.contributed.cpu().numpy().copy()
    # the same render again, this time with the blend loop's own flag
    n = len(g)
    flag = torch.zeros(n, dtype=torch.uint8, device="cuda")
    img = torch.empty_like(out.image)
    ft = torch.empty_like(out.final_t)
    nc = torch.empty_like(out.n_contrib)
    ke = torch.empty_like(out.k_eff_tiles)
    ck = torch.empty_like(out.ckpt)
    cm = torch.empty_like(out.ckpt_mask)
    work = torch.empty_like(out.work)
    st = torch.empty(_lib.STATUS_WORDS, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    assert L.ss_status_reset(P(st), stream_handle()) == 0
    rc = L.ss_blend_forward(ctypes.byref(out.camera.to_ss()), ctypes.byref(out.opts.to_ss()),
                            ctypes.byref(out.splats.ss()), ctypes.byref(out.bins.ss()), P(img),
                            P(ft), P(nc), None, P(ke), P(flag), P(ck), None, P(cm), P(work),
                            out.work_capacity, P(st), stream_handle())
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(img, out.image)
    np.testing.assert_array_equal(lazy, flag.cpu().numpy().astype(bool))
    assert lazy.sum() > 0


@pytest.mark.parametrize("offset", [0, 1, 3])
def test_check_finite_finds_every_position(offset):
    """ss_check_finite over unaligned views and every element class (16-byte
    body, scalar tail): a single NaN / Inf anywhere is reported, zeros and
    non-zeros are told apart."""
    _need_gpu()
    from paper_2410_00486_b200.rasterizer import finite_flags
    base = torch.ones(100003 + offset, device="cuda")
    t = base[offset:]
    assert finite_flags([t], extra_nonzero=True) == [True, True]
    for pos in (0, 5, 4097, len(t) - 1):
        for bad in (float("nan"), float("inf"), -float("inf")):
            u = t.clone()
            u[pos] = bad
            assert finite_flags([u, t]) == [False, True]
    z = torch.zeros(77, device="cuda")
    assert finite_flags([z, t], extra_nonzero=True) == [True, True, False, True]


def test_adam_step_rechecks_only_modified_gradients():
    """adam_step skips the reduction for gradients backward_splatwise's eager
    check passed, but a tensor modified in place since (a NaN written into
    it) is checked again and raises the reference's error
    (optimizer.py:111-113)."""
    _need_gpu()
    ss, g, cam = _scene(n=5000, seed=12)
    opts = ss.RasterOpts(sh_degree=0)
    tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(__import__(
        "paper_2410_00486_b200.scene", fromlist=["survey_scene"]).survey_scene(5000, 13)),
        cam, opts).image
    st = ss.AdamState.for_map(g)
    out = ss.rasterize_forward(g, cam, opts)
    lb = ss.compute_losses(out.image, tgt, g.opacity_logits)
    gr = ss.backward_splatwise(out, lb.grad_image)
    assert gr.known_finite("position", gr.position)[0]
    gr.opacity_logit += lb.grad_opacity_logit          # in place: version bumps
    assert not gr.known_finite("opacity_logit", gr.opacity_logit)[0]
    ss.adam_step(g, gr, st)                            # re-checks opacity only: passes
    out = ss.rasterize_forward(g, cam, opts)
    lb = ss.compute_losses(out.image, tgt, g.opacity_logits)
    gr = ss.backward_splatwise(out, lb.grad_image)
    gr.position[3, 1] = float("nan")
    before = g.positions.clone()
    with pytest.raises(FloatingPointError, match="position"):
        ss.adam_step(g, gr, st)
    assert torch.equal(before, g.positions)


def test_backward_clear_ahead_equals_backward_splat():
    """ss_backward_clear + ss_backward_splat_ex(SS_BWD_SKIP_CLEAR) -- the
    engine's split, the clear on a second stream -- gives the rows
    ss_backward_splat gives whatever the buffer held before (up to the order
    of the per-tile red.add rows); bad flags / column counts are rejected."""
    _need_gpu()
    from paper_2410_00486_b200 import _lib
    from paper_2410_00486_b200.rasterizer import P, screen_space_grads, stream_handle
    ss, g, cam = _scene(seed=14)
    opts = ss.RasterOpts(sh_degree=0)
    out = ss.rasterize_forward(g, cam, opts)
    gi = torch.randn_like(out.image)
    want = screen_space_grads(out, gi)
    n = out.n_primitives
    L = _lib.lib()
    cm, op = out.camera.to_ss(), out.opts.to_ss()
    g2d = torch.full((n, 9), float("nan"), device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        assert L.ss_backward_schedule(ctypes.byref(cm), P(out.k_eff_tiles), P(out.work),
                                      out.work_capacity, P(out.status), stream_handle()) == 0
        assert L.ss_backward_clear(n, 9, P(g2d), None, P(out.status), stream_handle()) == 0
    torch.cuda.current_stream().wait_stream(side)
    args = (ctypes.byref(cm), ctypes.byref(op), ctypes.byref(out.splats.ss()),
            ctypes.byref(out.bins.ss()), P(out.image), P(gi), None, P(out.depth), None,
            P(out.n_contrib), P(out.k_eff_tiles), P(out.ckpt), P(out.ckpt_depth),
            P(out.ckpt_mask), P(out.work), out.work_capacity, n, P(g2d), None, P(out.status))
    assert L.ss_backward_splat_ex(*args, 2, stream_handle()) == _lib.SS_EINVAL
    assert L.ss_backward_splat_ex(*args, _lib.SS_BWD_SKIP_CLEAR, stream_handle()) == 0
    torch.cuda.synchronize()
    assert torch.isfinite(g2d).all()
    scale = want.abs().amax(dim=0)
    assert ((g2d - want).abs() <= 1e-5 * scale + 1e-30).all()
    assert L.ss_backward_clear(n, 8, P(g2d), None, P(out.status), None) == _lib.SS_EINVAL


@pytest.mark.parametrize("depth", [False, True])
def test_warp_forward_bit_identical_to_cta_forward(depth):
    """The per-warp forward (default) and the CTA-batched forward (taken when
    the blend loop's contributed flags are asked for) write the same image,
    transmittance, n_contrib, k_eff, depth, checkpoints and blend masks, bit
    for bit, at a scene with long tile lists (many buckets per tile)."""
    _need_gpu()
    from paper_2410_00486_b200 import _lib
    from paper_2410_00486_b200.rasterizer import P, stream_handle
    ss, g, cam = _scene(n=30000, seed=15)
    out = ss.rasterize_forward(g, cam, ss.RasterOpts(sh_degree=0, with_depth=depth))
    assert int(out.k_eff_tiles.max()) > 64
    L = _lib.lib()
    res = []
    for flag in (None, torch.zeros(len(g), dtype=torch.uint8, device="cuda")):
        bufs = dict(img=torch.empty_like(out.image), ft=torch.empty_like(out.final_t),
                    nc=torch.empty_like(out.n_contrib), ke=torch.empty_like(out.k_eff_tiles),
                    ck=torch.full_like(out.ckpt, -7.0),
                    cm=torch.full_like(out.ckpt_mask, 0x5A5A5A5A),
                    work=torch.empty_like(out.work))
        if depth:
            bufs["d"] = torch.empty_like(out.depth)
            bufs["cd"] = torch.full_like(out.ckpt_depth, -7.0)
        st = torch.empty(_lib.STATUS_WORDS, dtype=torch.int64, device="cuda")
        assert L.ss_status_reset(P(st), stream_handle()) == 0
        rc = L.ss_blend_forward(ctypes.byref(out.camera.to_ss()), ctypes.byref(out.opts.to_ss()),
                                ctypes.byref(out.splats.ss()), ctypes.byref(out.bins.ss()),
                                P(bufs["img"]), P(bufs["ft"]), P(bufs["nc"]),
                                P(bufs.get("d")), P(bufs["ke"]), P(flag), P(bufs["ck"]),
                                P(bufs.get("cd")), P(bufs["cm"]), P(bufs["work"]),
                                out.work_capacity, P(st), stream_handle())
        assert rc == 0
        torch.cuda.synchronize()
        res.append(bufs)
    a, b = res
    for k in a:
        if k == "work":
            continue  # same entries, order of the tiles' appends differs
        assert torch.equal(a[k], b[k]), k
