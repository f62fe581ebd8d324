"""CPU parity oracle for the splatstream mapping hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package, and only as the checker or the timed CPU baseline.  The product
package ``paper_2410_00486_b200`` never imports it.

It restates the reference (``/root/reference/pkg/src/splatstream``) in
float64, the reference trainer's working dtype (``rasterizer/api.py:50``):
the per-primitive and per-tile arithmetic lives in ``splat_oracle.c``
(compiled by ``oracle/Makefile``); this module is the numpy orchestration
around it, following the reference's own call structure:

=========================  ============================================
oracle function            reference (file:line)
=========================  ============================================
``project``                ``rasterizer/projection.py:73-163``
``tile_index``             ``rasterizer/tiles.py:29-65``
``forward``                ``rasterizer/api.py:118-206``, ``kernels.py:14-152``
``replay``                 ``rasterizer/api.py:340-368``, ``kernels.py:155-178``
``backward_splat``         ``rasterizer/api.py:275-337``, ``kernels.py:271-373``
``backward_pixel``         ``rasterizer/api.py:227-272``, ``kernels.py:181-268``
``chain``                  ``rasterizer/projection.py:200-325``, ``api.py:217-224``
``losses``                 ``losses.py:198-228``
``adam``                   ``optimizer.py:101-133``
``accumulate_grad_stats``  ``densify.py:86-100``
``densify_and_prune``      ``densify.py:103-173``
``resize_for_densify``     ``optimizer.py:136-146``
``iteration``              ``trainer.py:180-215`` (``_Trainer.train_one``)
=========================  ============================================

Builder-defined extensions (absent from the
reference, so "parity unpinned" against it): the depth channel
(``with_depth``), ``opacity_reset`` and the multi-view gradient sum
(``multiview_grads``).

The oracle is pinned against golden vectors produced by the reference
itself (``tests/golden/make_golden.py``; checked by
``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsplat_oracle.so")
_lib = None

F64P = ctypes.POINTER(ctypes.c_double)
F32P = ctypes.POINTER(ctypes.c_float)
I64P = ctypes.POINTER(ctypes.c_int64)
I32P = ctypes.POINTER(ctypes.c_int32)
U8P = ctypes.POINTER(ctypes.c_uint8)
I64 = ctypes.c_int64
INT = ctypes.c_int
DBL = ctypes.c_double
VP = ctypes.c_void_p


def build() -> str:
    """Compile the C restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_project.restype = I64
        L.orc_project.argtypes = [I64, VP, VP, VP, VP, VP, VP, INT, DBL, DBL, DBL,
                                  VP, VP, VP, VP, VP, VP, VP, VP, VP]
        L.orc_tile_rects_f64.restype = I64
        L.orc_tile_rects_f64.argtypes = [I64, VP, VP, INT, I64, I64, VP]
        L.orc_tile_rects_f32.restype = I64
        L.orc_tile_rects_f32.argtypes = [I64, VP, VP, INT, I64, I64, VP]
        L.orc_tile_sort.restype = None
        L.orc_tile_sort.argtypes = [I64, VP, VP, I64, I64, I64, VP, VP]
        L.orc_forward.restype = None
        L.orc_forward.argtypes = [VP, VP, I64, VP, VP, VP, VP, VP, VP, VP, INT, INT, INT, INT,
                                  DBL, DBL, DBL, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, DBL, VP]
        L.orc_replay.restype = None
        L.orc_replay.argtypes = [VP, I64, I64, I64, VP, VP, VP, VP, VP, INT, INT, INT, INT,
                                 DBL, DBL, DBL, VP]
        L.orc_backward_splat.restype = None
        L.orc_backward_splat.argtypes = [VP, VP, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP,
                                         INT, INT, INT, INT, DBL, DBL, VP, VP, VP, VP, VP,
                                         I64, VP]
        L.orc_backward_pixel.restype = None
        L.orc_backward_pixel.argtypes = [VP, VP, I64, VP, VP, VP, VP, VP, VP, VP, INT, INT,
                                         INT, DBL, DBL, VP, VP, VP, I64, VP]
        L.orc_loss.restype = None
        L.orc_loss.argtypes = [I64, I64, VP, VP, DBL, VP, VP]
        L.orc_chain.restype = None
        L.orc_chain.argtypes = [I64, VP, VP, VP, VP, VP, VP, INT, DBL, I64, VP, VP,
                                VP, VP, VP, VP, VP, VP]
        L.orc_adam_group.restype = None
        L.orc_adam_group.argtypes = [I64, VP, VP, VP, VP, DBL, I64, DBL, DBL, DBL]
        L.orc_normalize_rotations.restype = INT
        L.orc_normalize_rotations.argtypes = [I64, VP]
        L.orc_set_threads.restype = None
        L.orc_set_threads.argtypes = [INT]
        L.orc_get_threads.restype = INT
        L.orc_get_threads.argtypes = []
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def _p(a):
    """Raw pointer of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle buffers must be C-contiguous"
    return a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------------------- data

@dataclass
class OMap:
    """Float64 parameter store with the reference's field names (core.py:120-128)."""

    positions: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    sh: np.ndarray
    grad2d_accum: np.ndarray = None
    grad3d_accum: np.ndarray = None
    obs_count: np.ndarray = None

    def __post_init__(self):
        n = self.positions.shape[0]
        self.positions = _f64(self.positions).reshape(n, 3).copy()
        self.rotations = _f64(self.rotations).reshape(n, 4).copy()
        self.log_scales = _f64(self.log_scales).reshape(n, 3).copy()
        self.opacity_logits = _f64(self.opacity_logits).reshape(n).copy()
        self.sh = _f64(self.sh).reshape(n, 16, 3).copy()
        if self.grad2d_accum is None:
            self.grad2d_accum = np.zeros(n)
        if self.grad3d_accum is None:
            self.grad3d_accum = np.zeros((n, 3))
        if self.obs_count is None:
            self.obs_count = np.zeros(n, dtype=np.int64)

    def __len__(self):
        return self.positions.shape[0]

    def copy(self) -> "OMap":
        return OMap(self.positions.copy(), self.rotations.copy(), self.log_scales.copy(),
                    self.opacity_logits.copy(), self.sh.copy(), self.grad2d_accum.copy(),
                    self.grad3d_accum.copy(), self.obs_count.copy())

    def first_nonfinite_index(self):
        """core.py:231-241."""
        bad = ~(np.isfinite(self.positions).all(1) & np.isfinite(self.rotations).all(1)
                & np.isfinite(self.log_scales).all(1) & np.isfinite(self.opacity_logits)
                & np.isfinite(self.sh).all(axis=(1, 2)))
        idx = np.flatnonzero(bad)
        return int(idx[0]) if idx.size else None


def cam_array(cam) -> np.ndarray:
    """Pack a camera (fx, fy, cx, cy, width, height, R, t) for the C side."""
    R = np.asarray(cam.R, dtype=np.float64).reshape(3, 3)
    t = np.asarray(cam.t, dtype=np.float64).reshape(3)
    centre = -R.T @ t
    return np.concatenate([[cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height],
                           R.reshape(9), t, centre]).astype(np.float64)


@dataclass
class OProjection:
    map_index: np.ndarray
    t_cam: np.ndarray
    depth: np.ndarray
    mean2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    radius: np.ndarray
    sigma: np.ndarray
    rgb: np.ndarray
    rgb_active: np.ndarray
    sh_degree: int = 3

    def __len__(self):
        return self.map_index.shape[0]


@dataclass
class OTileIndex:
    tile_size: int
    tiles_x: int
    tiles_y: int
    pair_splat: np.ndarray
    tile_range: np.ndarray
    active_tiles: np.ndarray

    def tile_origin(self, tile_id):
        ty, tx = divmod(int(tile_id), self.tiles_x)
        return tx * self.tile_size, ty * self.tile_size


@dataclass
class ORender:
    image: np.ndarray
    acc_rgb: np.ndarray
    final_t: np.ndarray
    n_contrib: np.ndarray
    proj: OProjection
    tile_index: OTileIndex
    k_eff: np.ndarray
    ckpt_flat: np.ndarray
    ckpt_off: np.ndarray
    contributed: np.ndarray
    m_cut: np.ndarray
    width: int
    height: int
    bucket: int
    t_min: float
    alpha_min: float
    alpha_max: float
    n_primitives: int
    depth: np.ndarray | None = None
    extra: dict = field(default_factory=dict)

    @property
    def alpha(self):
        """Builder extension A15: alpha = 1 - final_T (kernels.py:102)."""
        return 1.0 - self.final_t

    def checkpoints(self, stride=None):
        """Per active tile (nb, npx, stride) views, nb = ceil(k_eff / bucket)
        as in api.py:180-185."""
        st = stride or (5 if self.depth is not None else 4)
        out = []
        ti = self.tile_index
        for a, tid in enumerate(ti.active_tiles):
            x0, y0 = ti.tile_origin(tid)
            tw = min(ti.tile_size, self.width - x0)
            th = min(ti.tile_size, self.height - y0)
            nb = (int(self.k_eff[a]) + self.bucket - 1) // self.bucket
            o = int(self.ckpt_off[a])
            out.append(self.ckpt_flat[o:o + nb * tw * th * st].reshape(nb, tw * th, st))
        return out


@dataclass
class OGrads:
    position: np.ndarray
    rotation: np.ndarray
    log_scale: np.ndarray
    opacity_logit: np.ndarray
    sh: np.ndarray
    pos2d_grad_norm: np.ndarray
    contributed: np.ndarray

    def __len__(self):
        return self.position.shape[0]

    def validate_finite(self):
        """api.py:74-79."""
        for name in ("position", "rotation", "log_scale", "opacity_logit", "sh"):
            if not np.isfinite(getattr(self, name)).all():
                raise FloatingPointError(f"non-finite gradient in {name}")
        return self

    def __add__(self, other: "OGrads") -> "OGrads":
        return OGrads(self.position + other.position, self.rotation + other.rotation,
                      self.log_scale + other.log_scale, self.opacity_logit + other.opacity_logit,
                      self.sh + other.sh, self.pos2d_grad_norm + other.pos2d_grad_norm,
                      self.contributed | other.contributed)


@dataclass
class OLoss:
    l1: float
    ssim_loss: float
    rendered: float
    opacity_reg: float
    total: float
    grad_image: np.ndarray
    grad_opacity_logit: np.ndarray


# ---------------------------------------------------------------------- projection

def project(gmap: OMap, cam, sh_degree=3, near=0.01, dilation=0.3, alpha_min=1.0 / 255.0):
    """project_map (projection.py:73-163); rows compacted by map index."""
    n = len(gmap)
    c = cam_array(cam)
    vis = np.zeros(n, dtype=np.uint8)
    t_cam = np.zeros((n, 3))
    mean2d = np.zeros((n, 2))
    cov2d = np.zeros((n, 3))
    conic = np.zeros((n, 3))
    radius = np.zeros(n)
    sigma = np.zeros(n)
    rgb = np.zeros((n, 3))
    act = np.zeros((n, 3), dtype=np.uint8)
    sh = _f64(gmap.sh)
    rc = lib().orc_project(n, _p(gmap.positions), _p(gmap.rotations), _p(gmap.log_scales),
                           _p(gmap.opacity_logits), _p(sh), _p(c), int(sh_degree), near,
                           dilation, alpha_min, _p(vis), _p(t_cam), _p(mean2d), _p(cov2d),
                           _p(conic), _p(radius), _p(sigma), _p(rgb), _p(act))
    if rc < 0:
        raise ValueError(f"zero-norm quaternion at primitive {-rc - 1}")
    idx = np.flatnonzero(vis).astype(np.int32)
    return OProjection(map_index=idx, t_cam=t_cam[idx], depth=t_cam[idx, 2].copy(),
                       mean2d=mean2d[idx], cov2d=cov2d[idx], conic=conic[idx],
                       radius=radius[idx], sigma=sigma[idx], rgb=rgb[idx],
                       rgb_active=act[idx].astype(bool), sh_degree=sh_degree)


def m_cut_of(sigma, alpha_min=1.0 / 255.0):
    """api.py:150-151."""
    with np.errstate(divide="ignore"):
        return 2.0 * (np.log(np.asarray(sigma, np.float64)) - np.log(alpha_min))


# --------------------------------------------------------------------------- tiles

def tile_index(mean2d, radius, depth, width, height, tile=16) -> OTileIndex:
    """build_tile_index (tiles.py:29-65).  The rectangle arithmetic keeps the
    dtype of ``mean2d``/``radius`` (float32 projections stay float32, as numpy
    does in the reference), so a GPU float32 projection can be fed here for
    a bit-exact stage-wise comparison."""
    tiles_x = (width + tile - 1) // tile
    tiles_y = (height + tile - 1) // tile
    n_tiles = tiles_x * tiles_y
    m = int(np.asarray(radius).shape[0])
    if m == 0:
        return OTileIndex(tile, tiles_x, tiles_y, np.zeros(0, np.int32),
                          np.zeros(n_tiles + 1, np.int64), np.zeros(0, np.int64))
    rect = np.zeros((m, 4), dtype=np.int64)
    if np.asarray(mean2d).dtype == np.float32:
        mm = np.ascontiguousarray(mean2d, np.float32)
        rr = np.ascontiguousarray(radius, np.float32)
        total = lib().orc_tile_rects_f32(m, _p(mm), _p(rr), tile, tiles_x, tiles_y, _p(rect))
    else:
        mm = _f64(mean2d)
        rr = _f64(radius)
        total = lib().orc_tile_rects_f64(m, _p(mm), _p(rr), tile, tiles_x, tiles_y, _p(rect))
    dd = _f64(depth)
    pair = np.zeros(max(total, 1), dtype=np.int32)
    rng = np.zeros(n_tiles + 1, dtype=np.int64)
    lib().orc_tile_sort(m, _p(rect), _p(dd), tiles_x, n_tiles, total, _p(pair), _p(rng))
    active = np.flatnonzero(rng[1:] > rng[:-1]).astype(np.int64)
    return OTileIndex(tile, tiles_x, tiles_y, pair[:total].copy(), rng, active)


# ------------------------------------------------------------------------- forward

def forward(proj: OProjection, ti: OTileIndex, width, height, n_primitives, bucket=32,
            t_min=1e-4, alpha_min=1.0 / 255.0, alpha_max=0.99, background=(0.0, 0.0, 0.0),
            with_depth=False, m_cut=None, with_checkpoints=True,
            threshold_band=None) -> ORender:
    """rasterize_forward's blend stage (api.py:135-206) over forward_tile.

    ``threshold_band`` (parity support): also flag, per pixel, whether any
    of its (pixel, splat) evaluations lies within that relative band of the
    m_cut / alpha_min / t_min decisions (``extra["threshold_px"]``), i.e.
    where a float32 evaluation of the same inputs may decide differently."""
    W, H, ts = int(width), int(height), ti.tile_size
    bg = _f64(background).reshape(3)
    image = np.empty((H, W, 3))
    image[:] = bg
    acc = np.zeros((H, W, 3))
    final_t = np.ones((H, W))
    n_contrib = np.zeros((H, W), dtype=np.int32)
    m = len(proj)
    contributed_proj = np.zeros(max(m, 1), dtype=np.uint8)
    if m_cut is None:
        m_cut = m_cut_of(proj.sigma, alpha_min)
    m_cut = _f64(m_cut)
    active = np.ascontiguousarray(ti.active_tiles, np.int64)
    A = active.shape[0]
    stride = 5 if with_depth else 4
    lens = ti.tile_range[active + 1] - ti.tile_range[active]
    tx0 = (active % ti.tiles_x) * ts
    ty0 = (active // ti.tiles_x) * ts
    npx = np.minimum(ts, W - tx0) * np.minimum(ts, H - ty0)
    sizes = ((lens + bucket - 1) // bucket) * npx * stride if with_checkpoints else np.zeros(A, np.int64)
    ckpt_off = np.zeros(A + 1, dtype=np.int64)
    np.cumsum(sizes, out=ckpt_off[1:])
    ckpt = np.zeros(max(int(ckpt_off[-1]), 1)) if with_checkpoints else None
    k_eff = np.zeros(A, dtype=np.int64)
    depth = _f64(proj.depth) if with_depth else None
    dimg = np.zeros((H, W)) if with_depth else None
    thr = np.zeros((H, W), dtype=np.uint8) if threshold_band is not None else None
    lib().orc_forward(_p(np.ascontiguousarray(ti.pair_splat, np.int32)), _p(ti.tile_range), A,
                      _p(active), _p(_f64(proj.mean2d)), _p(_f64(proj.conic)), _p(_f64(proj.rgb)),
                      _p(_f64(proj.sigma)), _p(m_cut), _p(depth), W, H, ts, bucket, t_min,
                      alpha_min, alpha_max, _p(bg), _p(image), _p(acc), _p(final_t),
                      _p(n_contrib), _p(k_eff), _p(contributed_proj), _p(ckpt), _p(ckpt_off),
                      _p(dimg), float(threshold_band or 0.0), _p(thr))
    contributed = np.zeros(n_primitives, dtype=bool)
    if m:
        contributed[proj.map_index[contributed_proj[:m].astype(bool)]] = True
    r = ORender(image=image, acc_rgb=acc, final_t=final_t, n_contrib=n_contrib, proj=proj,
                tile_index=ti, k_eff=k_eff, ckpt_flat=ckpt, ckpt_off=ckpt_off,
                contributed=contributed, m_cut=m_cut, width=W, height=H, bucket=bucket,
                t_min=t_min, alpha_min=alpha_min, alpha_max=alpha_max,
                n_primitives=n_primitives, depth=dimg)
    if thr is not None:
        r.extra["threshold_px"] = thr.astype(bool)
    return r


def rasterize(gmap: OMap, cam, sh_degree=3, tile=16, bucket=32, t_min=1e-4,
              alpha_min=1.0 / 255.0, alpha_max=0.99, background=(0.0, 0.0, 0.0), near=0.01,
              dilation=0.3, with_depth=False, with_checkpoints=True) -> ORender:
    """rasterize_forward (api.py:118-206)."""
    bad = gmap.first_nonfinite_index()
    if bad is not None:
        raise ValueError(f"non-finite parameter in primitive {bad}")
    proj = project(gmap, cam, sh_degree, near, dilation, alpha_min)
    ti = tile_index(proj.mean2d, proj.radius, proj.depth, cam.width, cam.height, tile)
    r = forward(proj, ti, cam.width, cam.height, len(gmap), bucket, t_min, alpha_min, alpha_max,
                background, with_depth, with_checkpoints=with_checkpoints)
    r.extra["dilation"] = dilation
    return r


def replay(render: ORender, tile_pos: int, from_bucket: int, n_positions=None):
    """replay_pixel_states (api.py:340-368): returns (T, rgb) after
    advancing a checkpoint."""
    ti = render.tile_index
    tid = int(ti.active_tiles[tile_pos])
    ke = int(render.k_eff[tile_pos])
    x0, y0 = ti.tile_origin(tid)
    tw = min(ti.tile_size, render.width - x0)
    th = min(ti.tile_size, render.height - y0)
    ck = render.checkpoints(4)[tile_pos][from_bucket] if render.depth is None else \
        render.checkpoints(5)[tile_pos][from_bucket][:, :4]
    state = np.ascontiguousarray(ck, dtype=np.float64).copy()
    pos_from = from_bucket * render.bucket
    pos_to = ke if n_positions is None else min(ke, pos_from + n_positions)
    p = render.proj
    lib().orc_replay(_p(np.ascontiguousarray(ti.pair_splat, np.int32)), int(ti.tile_range[tid]),
                     pos_from, pos_to, _p(_f64(p.mean2d)), _p(_f64(p.conic)), _p(_f64(p.rgb)),
                     _p(_f64(p.sigma)), _p(render.m_cut), x0, y0, tw, th, render.t_min,
                     render.alpha_min, render.alpha_max, _p(state))
    return state[:, 0].copy(), state[:, 1:4].copy()


# ------------------------------------------------------------------------ backward

def _check_grad_image(render, grad_image):
    if grad_image.shape != render.image.shape:
        raise ValueError(f"grad_image shape {grad_image.shape} does not match "
                         f"rendered image shape {render.image.shape}")
    return _f64(grad_image)


def backward_splat(render: ORender, grad_image, grad_depth=None) -> np.ndarray:
    """Splat-wise backward up to g2d (api.py:275-336).  Returns (M, 9), or
    (M, 10) with the depth extension: [rgb3, mean2d2, conic3, opacity, z]."""
    if render.ckpt_flat is None:
        raise RuntimeError("render output has no checkpoints; re-run rasterize_forward "
                           "with with_checkpoints=True to use the splat-wise backward")
    g = _check_grad_image(render, grad_image)
    ti, p = render.tile_index, render.proj
    with_depth = render.depth is not None
    ncol = 10 if with_depth else 9
    g2d = np.zeros((max(len(p), 1), ncol))
    gd = _f64(grad_depth) if (with_depth and grad_depth is not None) else (
        np.zeros((render.height, render.width)) if with_depth else None)
    lib().orc_backward_splat(
        _p(np.ascontiguousarray(ti.pair_splat, np.int32)), _p(ti.tile_range),
        ti.active_tiles.shape[0], _p(np.ascontiguousarray(ti.active_tiles, np.int64)),
        _p(render.k_eff), _p(render.ckpt_flat), _p(render.ckpt_off), _p(_f64(p.mean2d)),
        _p(_f64(p.conic)), _p(_f64(p.rgb)), _p(_f64(p.sigma)), _p(render.m_cut),
        _p(_f64(p.depth) if with_depth else None), render.width, render.height, ti.tile_size,
        render.bucket, render.alpha_min, render.alpha_max, _p(g), _p(_f64(render.image)),
        _p(render.n_contrib), _p(gd), _p(render.depth), len(p), _p(g2d))
    return g2d[:len(p)]


def backward_pixel(render: ORender, grad_image) -> np.ndarray:
    """Pixel-wise backward up to g2d (api.py:227-271)."""
    g = _check_grad_image(render, grad_image)
    ti, p = render.tile_index, render.proj
    g2d = np.zeros((max(len(p), 1), 9))
    lib().orc_backward_pixel(
        _p(np.ascontiguousarray(ti.pair_splat, np.int32)), _p(ti.tile_range),
        ti.active_tiles.shape[0], _p(np.ascontiguousarray(ti.active_tiles, np.int64)),
        _p(render.k_eff), _p(_f64(p.mean2d)), _p(_f64(p.conic)), _p(_f64(p.rgb)),
        _p(_f64(p.sigma)), _p(render.m_cut), render.width, render.height, ti.tile_size,
        render.alpha_min, render.alpha_max, _p(g), _p(_f64(render.image)),
        _p(render.n_contrib), len(p), _p(g2d))
    return g2d[:len(p)]


def chain(gmap: OMap, cam, proj: OProjection, g2d, contributed, dilation=0.3) -> OGrads:
    """chain_backward (projection.py:200-299) + _finish_backward (api.py:217-224).
    A 10th g2d column (depth extension) chains into the camera-frame z."""
    n = len(gmap)
    g2d = _f64(g2d)
    m = len(proj)
    gp = np.zeros((n, 3)); gr = np.zeros((n, 4)); gl = np.zeros((n, 3)); go = np.zeros(n)
    gs = np.zeros((n, 16, 3)); pn = np.zeros(n)
    mi = np.ascontiguousarray(proj.map_index, np.int64)
    lib().orc_chain(n, _p(gmap.positions), _p(gmap.rotations), _p(gmap.log_scales),
                    _p(gmap.opacity_logits), _p(_f64(gmap.sh)), _p(cam_array(cam)),
                    int(proj.sh_degree), dilation, m, _p(mi), _p(np.ascontiguousarray(g2d[:, :9])),
                    _p(gp), _p(gr), _p(gl), _p(go), _p(gs), _p(pn))
    if g2d.shape[1] == 10 and m:
        # depth extension: z = (R p + t)_z, so dL/dp += g_z * R[2, :]
        R = np.asarray(cam.R, np.float64).reshape(3, 3)
        gp[mi] += g2d[:, 9:10] * R[2][None, :]
    return OGrads(gp, gr, gl, go, gs, pn, np.asarray(contributed, bool).copy()).validate_finite()


# --------------------------------------------------------------------------- loss

def losses(rendered, target, opacity_logits, lambda_ssim=0.2, lambda_o=0.001) -> OLoss:
    """compute_losses (losses.py:198-228)."""
    x = _f64(rendered)
    y = _f64(target)
    if x.shape != y.shape:
        raise ValueError(f"image shapes differ: {x.shape} vs {y.shape}")
    H, W = x.shape[0], x.shape[1]
    out = np.zeros(2)
    grad = np.zeros_like(x)
    lib().orc_loss(H, W, _p(x), _p(y), float(lambda_ssim), _p(out), _p(grad))
    l1 = float(out[0])
    ssim_loss = 1.0 - float(out[1]) if lambda_ssim != 0.0 else 0.0
    rendered_val = (1.0 - lambda_ssim) * l1 + lambda_ssim * ssim_loss
    logits = _f64(opacity_logits)
    n = logits.size
    sig = 1.0 / (1.0 + np.exp(-logits)) if n else np.zeros(0)
    reg = float(np.mean(np.abs(sig))) if n else 0.0
    reg_grad = np.sign(sig) / n if n else np.zeros(0)
    return OLoss(l1=l1, ssim_loss=ssim_loss, rendered=rendered_val, opacity_reg=reg,
                 total=rendered_val + lambda_o * reg, grad_image=grad,
                 grad_opacity_logit=lambda_o * reg_grad * sig * (1.0 - sig))


def depth_loss(depth, target_depth, valid=None):
    """Builder-defined depth term (the reference has no
    depth): mean |D - D*| over valid target pixels, grad sign(D - D*)/n."""
    d = _f64(depth) - _f64(target_depth)
    mask = np.ones_like(d, bool) if valid is None else np.asarray(valid, bool)
    n = max(int(mask.sum()), 1)
    return float(np.abs(d[mask]).sum() / n), np.where(mask, np.sign(d), 0.0) / n


# ---------------------------------------------------------------------- optimizer

PARAM_SHAPES = {"position": (3,), "rotation": (4,), "log_scale": (3,), "opacity_logit": (),
                "sh_dc": (1, 3), "sh_rest": (15, 3)}


@dataclass
class OAdam:
    """AdamState (optimizer.py:29-76), float64 moments keyed like the reference."""

    lrs: dict = field(default_factory=lambda: dict(
        position=1.6e-4, position_final=1.6e-6, sh_dc=2.5e-3, sh_rest=1.25e-4,
        opacity_logit=5e-2, log_scale=5e-3, rotation=1e-3))
    horizon: int = 30000
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    step_count: int = 0
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)

    @classmethod
    def for_map(cls, gmap, horizon=30000):
        st = cls(horizon=horizon)
        n = len(gmap)
        for k, shp in PARAM_SHAPES.items():
            st.m[k] = np.zeros((n,) + shp)
            st.v[k] = np.zeros((n,) + shp)
        return st

    def copy(self):
        return OAdam(dict(self.lrs), self.horizon, self.beta1, self.beta2, self.eps,
                     self.step_count, {k: v.copy() for k, v in self.m.items()},
                     {k: v.copy() for k, v in self.v.items()})

    def position_lr(self):
        t = min(self.step_count / max(self.horizon, 1), 1.0)
        lr0, lr1 = self.lrs["position"], self.lrs["position_final"]
        return float(lr0 * (lr1 / lr0) ** t)

    def rate_for(self, name):
        return self.position_lr() if name == "position" else self.lrs[name]


def adam(gmap: OMap, grads: OGrads, st: OAdam):
    """adam_step (optimizer.py:101-133), in place."""
    if len(grads) != len(gmap):
        raise ValueError(f"gradient length {len(grads)} does not match map length {len(gmap)}")
    gv = {"position": grads.position, "rotation": grads.rotation, "log_scale": grads.log_scale,
          "opacity_logit": grads.opacity_logit, "sh_dc": grads.sh[:, :1, :],
          "sh_rest": grads.sh[:, 1:, :]}
    for k, g in gv.items():
        if not np.isfinite(g).all():
            raise FloatingPointError(f"non-finite gradient for parameter '{k}'")
    st.step_count += 1
    sh_dc = np.ascontiguousarray(gmap.sh[:, :1, :])
    sh_rest = np.ascontiguousarray(gmap.sh[:, 1:, :])
    pv = {"position": gmap.positions, "rotation": gmap.rotations, "log_scale": gmap.log_scales,
          "opacity_logit": gmap.opacity_logits, "sh_dc": sh_dc, "sh_rest": sh_rest}
    for k, p in pv.items():
        g = np.ascontiguousarray(gv[k], np.float64)
        lib().orc_adam_group(p.size, _p(p), _p(g), _p(st.m[k]), _p(st.v[k]), st.rate_for(k),
                             st.step_count, st.beta1, st.beta2, st.eps)
    gmap.sh[:, :1, :] = sh_dc
    gmap.sh[:, 1:, :] = sh_rest
    if lib().orc_normalize_rotations(len(gmap), _p(gmap.rotations)) != 0:
        raise ValueError("zero-norm quaternion in map")
    return gmap, st


def resize_for_densify(st: OAdam, survivors, n_new):
    """optimizer.py:136-146."""
    survivors = np.asarray(survivors, np.int64)
    for k, shp in PARAM_SHAPES.items():
        z = np.zeros((n_new,) + shp)
        st.m[k] = np.concatenate([st.m[k][survivors], z])
        st.v[k] = np.concatenate([st.v[k][survivors], z])
    return st


# ------------------------------------------------------------------------ densify

def accumulate_grad_stats(gmap: OMap, grads: OGrads):
    """densify.py:86-100."""
    if len(grads) != len(gmap):
        raise ValueError(f"gradient length {len(grads)} does not match map length {len(gmap)}")
    seen = grads.contributed
    gmap.grad2d_accum[seen] += grads.pos2d_grad_norm[seen]
    gmap.grad3d_accum[seen] += grads.position[seen]
    gmap.obs_count[seen] += 1
    return gmap


def _quat_rot(q):
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], 1)


def densify_masks(gmap: OMap, grad_threshold=0.001, prune_opacity=0.02,
                  split_scale_percentile=0.01, scene_extent=1.0):
    """The three masks of densify_and_prune (densify.py:110-117,148), float64."""
    counts = np.maximum(gmap.obs_count, 1)
    mean_norm = gmap.grad2d_accum / counts
    cand = (mean_norm > grad_threshold) & (gmap.obs_count > 0)
    max_scale = np.exp(gmap.log_scales).max(axis=1) if len(gmap) else np.zeros(0)
    small = cand & (max_scale <= split_scale_percentile * scene_extent)
    large = cand & ~small
    sig = np.empty(len(gmap))
    pos = gmap.opacity_logits >= 0
    sig[pos] = 1.0 / (1.0 + np.exp(-gmap.opacity_logits[pos]))
    ex = np.exp(gmap.opacity_logits[~pos])
    sig[~pos] = ex / (1.0 + ex)
    keep_old = ~large & (sig >= prune_opacity)
    return small, large, keep_old


def densify_and_prune(gmap: OMap, normals=None, rng=None, grad_threshold=0.001,
                      prune_opacity=0.02, split_scale_percentile=0.01, split_children=2,
                      split_scale_shrink=1.6, clone_step=0.01, scene_extent=1.0):
    """densify_and_prune (densify.py:103-173).  Split offsets use ``normals``
    ((n_split*children, 3) standard normals) when given, else draw them from
    ``rng.standard_normal`` exactly where the reference does (densify.py:137)."""
    counts = np.maximum(gmap.obs_count, 1)
    mean_g3d = gmap.grad3d_accum / counts[:, None]
    small, large, keep_old = densify_masks(gmap, grad_threshold, prune_opacity,
                                           split_scale_percentile, scene_extent)
    parts = []
    clone_idx = np.flatnonzero(small)
    if clone_idx.size:
        parts.append((gmap.positions[clone_idx] - clone_step * mean_g3d[clone_idx],
                      gmap.rotations[clone_idx], gmap.log_scales[clone_idx],
                      gmap.opacity_logits[clone_idx], gmap.sh[clone_idx]))
    split_idx = np.flatnonzero(large)
    if split_idx.size:
        rep = np.repeat(split_idx, split_children)
        if normals is None:
            if rng is None:
                rng = np.random.default_rng()
            normals = rng.standard_normal((rep.size, 3))
        local = np.asarray(normals, np.float64).reshape(rep.size, 3) * np.exp(gmap.log_scales[rep])
        R = _quat_rot(gmap.rotations[rep])
        parts.append((gmap.positions[rep] + np.einsum("nij,nj->ni", R, local),
                      gmap.rotations[rep], gmap.log_scales[rep] - np.log(split_scale_shrink),
                      gmap.opacity_logits[rep], gmap.sh[rep]))
    survivors = np.flatnonzero(keep_old)
    n_pruned = int(np.sum(~keep_old & ~large))
    if parts:
        cat = [np.concatenate([p[j] for p in parts]) for j in range(5)]
        fresh = 1.0 / (1.0 + np.exp(-cat[3])) >= prune_opacity
        cat = [c[fresh] for c in cat]
    else:
        cat = [np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
               np.zeros((0, 16, 3))]
    n_new = cat[0].shape[0]
    new = OMap(np.concatenate([gmap.positions[keep_old], cat[0]]),
               np.concatenate([gmap.rotations[keep_old], cat[1]]),
               np.concatenate([gmap.log_scales[keep_old], cat[2]]),
               np.concatenate([gmap.opacity_logits[keep_old], cat[3]]),
               np.concatenate([gmap.sh[keep_old], cat[4]]))
    return new, dict(survivors=survivors, n_new=n_new, n_cloned=int(clone_idx.size),
                     n_split=int(split_idx.size), n_pruned=n_pruned,
                     small=small, large=large, keep_old=keep_old)


def opacity_reset(gmap: OMap, st: OAdam | None = None, ceiling=0.01):
    """Builder-defined opacity reset (SURVEY 8a A16, 3DGS convention):
    logit <- logit(min(sigma, ceiling)); opacity moments zeroed."""
    sig = 1.0 / (1.0 + np.exp(-gmap.opacity_logits))
    new = np.minimum(sig, ceiling)
    gmap.opacity_logits = np.log(new) - np.log1p(-new)
    if st is not None and "opacity_logit" in st.m:
        st.m["opacity_logit"][:] = 0.0
        st.v["opacity_logit"][:] = 0.0
    return gmap


# ---------------------------------------------------------------------- iteration

def iteration(gmap: OMap, cam, target, st: OAdam, sh_degree=0, lambda_ssim=0.2,
              lambda_o=0.001, background=(0.0, 0.0, 0.0), keep=False):
    """One mapping iteration, the _Trainer.train_one sequence
    (trainer.py:199-208): forward -> losses -> splat-wise
    backward -> + opacity-reg grad -> adam -> grad stats.  In place on
    gmap/st; returns the loss breakdown (and intermediates with keep)."""
    r = rasterize(gmap, cam, sh_degree=sh_degree, background=background)
    lb = losses(r.image, target, gmap.opacity_logits, lambda_ssim, lambda_o)
    g2d = backward_splat(r, lb.grad_image)
    gr = chain(gmap, cam, r.proj, g2d, r.contributed)
    gr.opacity_logit = gr.opacity_logit + lb.grad_opacity_logit
    adam(gmap, gr, st)
    accumulate_grad_stats(gmap, gr)
    if keep:
        return lb, dict(render=r, g2d=g2d, grads=gr)
    return lb


def multiview_grads(gmap: OMap, cams, targets, sh_degree=0, lambda_ssim=0.2, lambda_o=0.001):
    """Builder-defined multi-view step: per-view ParamGrads
    summed, the opacity-regulariser gradient added once."""
    total = None
    losses_ = []
    for cam, tgt in zip(cams, targets):
        r = rasterize(gmap, cam, sh_degree=sh_degree)
        lb = losses(r.image, tgt, gmap.opacity_logits, lambda_ssim, lambda_o)
        g = chain(gmap, cam, r.proj, backward_splat(r, lb.grad_image), r.contributed)
        total = g if total is None else total + g
        losses_.append(lb)
    total.opacity_logit = total.opacity_logit + losses_[0].grad_opacity_logit
    return total, losses_


__all__ = [n for n in dir() if not n.startswith("_")]
_ = math


# ---------------------------------------------------------------- seeding

def seed_from_points(points, colors, scene_extent=1.0):
    """seed_from_points (densify.py:53-83): one isotropic primitive per point,
    scale = mean distance to the 3 nearest neighbours within the cloud
    (brute-force float64 kNN in chunks: the k + 1 smallest distances
    including the point itself, self dropped, as cKDTree.query(k=4)[:, 1:]),
    floored at 1e-4 (a lone point: 0.01 * scene_extent); identity rotation,
    opacity logit(0.1), DC colour (c - 0.5) / SH_C0."""
    p = np.asarray(points, np.float64).reshape(-1, 3)
    c = np.asarray(colors, np.float64).reshape(-1, 3)
    n = p.shape[0]
    if n == 0:
        return (np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                np.zeros((0, 16, 3)))
    if not np.isfinite(p).all():
        raise ValueError("non-finite point in seed cloud")
    if n == 1:
        md = np.array([0.01 * scene_extent])
    else:
        k = min(3, n - 1)
        md = np.empty(n)
        for a in range(0, n, 512):
            d2 = ((p[a:a + 512, None, :] - p[None, :, :]) ** 2).sum(-1)
            part = np.sqrt(np.partition(d2, k, axis=1)[:, :k + 1])
            part.sort(axis=1)
            md[a:a + 512] = part[:, 1:].mean(axis=1)
    ls = np.log(np.maximum(md, 1e-4))[:, None].repeat(3, axis=1)
    rot = np.zeros((n, 4))
    rot[:, 0] = 1.0
    op = np.full(n, np.log(0.1 / 0.9))
    sh = np.zeros((n, 16, 3))
    sh[:, 0, :] = (c - 0.5) / 0.28209479177387814
    return p.copy(), rot, ls, op, sh
