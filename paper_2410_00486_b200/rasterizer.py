"""Forward rendering and the splat-wise backward on B200.

Drop-in for ``splatstream.rasterizer`` (rasterizer/api.py:37-368): same
names (``RasterOpts``, ``RenderOutput``, ``ParamGrads``,
``rasterize_forward``, ``backward_splatwise``), same argument meaning and
error behaviour; outputs are float32 CUDA tensors.  All compute runs in
libss_b200.so (K1 preprocess, K2-K4b binning, K5 blend, K7 splat-wise
backward, K8 chain); this module only allocates buffers and sequences the
C-ABI calls on the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, errors
from ._lib import check, lib, traced
from .core import Camera, GaussianMap

G2D_COLS = 9
EAGER_CKPT_MAX_LIST = 1024  # api.py:23 -- the GPU always checkpoints in the forward pass


@dataclass
class RasterOpts:
    """api.py:37-52.  ``dtype`` and ``n_workers`` are accepted for drop-in
    compatibility; the B200 path always computes in float32 on the GPU."""

    tile_size: int = 16
    bucket_size: int = 32
    t_min: float = 1e-4
    alpha_min: float = 1.0 / 255.0
    alpha_max: float = 0.99
    background: tuple = (0.0, 0.0, 0.0)
    sh_degree: int = 3
    near: float = 0.01
    dilation: float = 0.3
    dtype: type = np.float32
    with_checkpoints: bool = True
    n_workers: int = 1
    with_depth: bool = False  # builder extension A15

    def to_ss(self) -> _lib.SSRasterOpts:
        if self.tile_size != 16 or self.bucket_size != 32:
            raise ValueError("the B200 kernels are specialised for tile_size=16, bucket_size=32")
        o = _lib.SSRasterOpts()
        o.tile_size, o.bucket_size = 16, 32
        o.t_min, o.alpha_min, o.alpha_max = self.t_min, self.alpha_min, self.alpha_max
        o.background[:] = [float(b) for b in self.background]
        o.sh_degree = int(self.sh_degree)
        o.near_plane, o.dilation = self.near, self.dilation
        o.with_depth = 1 if self.with_depth else 0
        return o


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def P(t):
    """Device pointer of a tensor (None for empty / missing)."""
    if t is None or t.numel() == 0:
        return None
    return ctypes.c_void_p(t.data_ptr())


@dataclass
class SplatBuffers:
    """Per-Gaussian K1 outputs (ss_splats)."""

    rec: torch.Tensor       # (n, 12) float32: SplatRec
    depth_key: torch.Tensor  # (n,) int32 (u32 bits)
    tiles: torch.Tensor     # (n,) int32
    rect: torch.Tensor      # (n, 2) int32
    flags: torch.Tensor     # (n,) uint8
    aux: torch.Tensor | None  # (n, 8) float32

    @classmethod
    def alloc(cls, n, dev, aux=True):
        return cls(torch.empty((n, 12), dtype=torch.float32, device=dev),
                   torch.empty(n, dtype=torch.int32, device=dev),
                   torch.empty(n, dtype=torch.int32, device=dev),
                   torch.empty((n, 2), dtype=torch.int32, device=dev),
                   torch.empty(n, dtype=torch.uint8, device=dev),
                   torch.empty((n, 8), dtype=torch.float32, device=dev) if aux else None)

    def ss(self):
        s = _lib.SSSplats()
        s.d_rec, s.d_depth_key, s.d_tiles = P(self.rec), P(self.depth_key), P(self.tiles)
        s.d_rect, s.d_flags, s.d_aux = P(self.rect), P(self.flags), P(self.aux)
        return s


@dataclass
class BinBuffers:
    """K2-K4b outputs (ss_bins)."""

    capacity: int
    pairs: torch.Tensor      # (capacity,) int32 Gaussian ids
    tile_start: torch.Tensor  # (T,)
    tile_end: torch.Tensor    # (T,)
    ckpt_base: torch.Tensor   # (T+1,)
    tile_order: torch.Tensor  # (T,) forward CTA -> tile, costliest first (identity at start)
    tile_cost: torch.Tensor   # (T,) last forward's per-tile cost (SM cycles)

    @classmethod
    def alloc(cls, cap, n_tiles, dev):
        i32 = dict(dtype=torch.int32, device=dev)
        return cls(cap, torch.empty(max(cap, 1), **i32), torch.empty(n_tiles, **i32),
                   torch.empty(n_tiles, **i32), torch.empty(n_tiles + 1, **i32),
                   torch.arange(n_tiles, **i32), torch.zeros(n_tiles, **i32))

    def ss(self):
        b = _lib.SSBins()
        b.pair_capacity = self.capacity
        b.d_pair_splat, b.d_tile_start = P(self.pairs), P(self.tile_start)
        b.d_tile_end, b.d_ckpt_base = P(self.tile_end), P(self.ckpt_base)
        if self.tile_order is not None and self.tile_order.numel() <= _lib.ORDER_MAX_TILES:
            b.d_tile_order, b.d_tile_cost = P(self.tile_order), P(self.tile_cost)
        return b


_CAP_HINT: dict = {}
# per (device, tile grid): the last forward's per-tile blend cost, which the
# next call's binning turns into the costliest-first CTA order (the forward's
# results do not depend on it; only its tail does)
_COST_HINT: dict = {}


def new_status(dev):
    st = torch.empty(_lib.STATUS_WORDS, dtype=torch.int64, device=dev)
    check(lib().ss_status_reset(P(st), stream_handle()), "ss_status_reset")
    return st


def finite_flags_device(tensors):
    """Device int32 flags (2 n): [t] = tensor t holds a non-finite value,
    [n + t] = it holds a non-zero value -- one ss_check_finite launch, no
    host read."""
    ts = [t.contiguous() if t.dtype == torch.float32 else t.float().contiguous()
          for t in tensors]
    n = len(ts)
    flags = torch.empty(2 * n, dtype=torch.int32, device=ts[0].device)
    ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() if t.numel() else None for t in ts])
    cnts = (ctypes.c_int64 * n)(*[t.numel() for t in ts])
    check(lib().ss_check_finite(n, ptrs, cnts, P(flags), stream_handle()), "ss_check_finite")
    return flags


def finite_flags(tensors, extra_nonzero=False):
    """[all(isfinite(t)) for t in tensors] (+ [any(t != 0)] per tensor with
    extra_nonzero) from one kernel and ONE host read."""
    if not tensors:
        return []
    h = finite_flags_device(tensors).cpu().tolist()
    n = len(tensors)
    out = [h[t] == 0 for t in range(n)]
    return out + ([h[n + t] != 0 for t in range(n)] if extra_nonzero else [])


def raise_param_errors(st_host):
    bad = int(st_host[_lib.ST_BAD_PARAM])
    if bad != _lib.INT64_MAX:
        raise ValueError(f"non-finite parameter in primitive {bad}")
    zq = int(st_host[_lib.ST_ZERO_QUAT])
    if zq != _lib.INT64_MAX:
        raise ValueError(f"zero-norm quaternion at primitive {zq}")


def bin_workspace(n, cap, n_tiles, dev):
    nbytes = int(lib().ss_bin_workspace_bytes(n, cap, n_tiles))
    return torch.empty(nbytes, dtype=torch.uint8, device=dev)


@dataclass
class Projection:
    """Reference-shaped view of the K1 output (projection.py:40-65), built
    on request: rows are the visible Gaussians in index order."""

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
    m_cut: np.ndarray
    sh_degree: int
    # device-side K1 outputs this view was built from (SplatBuffers, Camera,
    # GaussianMap, RasterOpts), so build_tile_index / chain_backward on a
    # Projection from project_map stay on the GPU
    _device: tuple | None = field(default=None, repr=False, compare=False)

    def __len__(self):
        return int(self.map_index.shape[0])


def _projection_from_splats(splats: SplatBuffers, sh_degree: int, dtype=np.float32) -> Projection:
    """Reference-shaped (compacted, host) view of the K1 output."""
    fl = splats.flags.cpu().numpy()
    vis = np.flatnonzero(fl & 1).astype(np.int32)
    rec = splats.rec.cpu().numpy()[vis]
    aux = splats.aux.cpu().numpy()[vis] if splats.aux is not None else None
    act = np.stack([(fl[vis] >> 1) & 1, (fl[vis] >> 2) & 1, (fl[vis] >> 3) & 1], 1)
    dt = np.dtype(dtype)
    c = (lambda a: None if a is None else np.ascontiguousarray(a, dtype=dt))
    return Projection(
        map_index=vis, t_cam=c(aux[:, 0:3]) if aux is not None else None,
        depth=c(rec[:, 7]), mean2d=c(rec[:, 0:2]),
        cov2d=c(aux[:, 3:6]) if aux is not None else None,
        conic=c(np.stack([rec[:, 2], 0.5 * rec[:, 3], rec[:, 4]], 1)),
        radius=c(aux[:, 6]) if aux is not None else None, sigma=c(rec[:, 5]), rgb=c(rec[:, 8:11]),
        rgb_active=act.astype(bool), m_cut=c(rec[:, 6]), sh_degree=sh_degree)


@dataclass
class TileIndex:
    """tiles.py:15-26 view; ``pair_splat`` holds projection-row indices like
    the reference (``pair_gaussian`` the Gaussian ids the kernels use)."""

    tile_size: int
    tiles_x: int
    tiles_y: int
    pair_splat: np.ndarray
    pair_gaussian: np.ndarray
    tile_range: np.ndarray
    active_tiles: np.ndarray

    def tile_origin(self, tile_id):
        ty, tx = divmod(int(tile_id), self.tiles_x)
        return tx * self.tile_size, ty * self.tile_size


@dataclass
class RenderOutput:
    """api.py:82-105 plus the device buffers the splat-wise backward reads."""

    image: torch.Tensor      # (H, W, 3)
    final_t: torch.Tensor    # (H, W)
    n_contrib: torch.Tensor  # (H, W) int32
    k_eff_tiles: torch.Tensor  # (T,) int32, per tile (all tiles)
    contributed_buf: torch.Tensor | None  # (N,) bool once derived (see `contributed`)
    opts: RasterOpts
    camera: Camera
    n_primitives: int
    gmap: GaussianMap
    splats: SplatBuffers
    bins: BinBuffers
    pair_count: int
    ckpt: torch.Tensor | None
    ckpt_depth: torch.Tensor | None
    ckpt_mask: torch.Tensor
    work: torch.Tensor
    work_capacity: int
    status: torch.Tensor
    depth: torch.Tensor | None = None
    _cache: dict = field(default_factory=dict)

    @property
    def contributed(self) -> torch.Tensor:
        """(N,) bool: Gaussians blended into at least one pixel (kernels.py:94-95),
        derived from the forward's blend masks on first use (one kernel)."""
        if self.contributed_buf is None:
            n = self.n_primitives
            dev = self.image.device
            buf = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
            check(lib().ss_contributed_from_masks(
                ctypes.byref(self.camera.to_ss()), ctypes.byref(self.bins.ss()),
                P(self.n_contrib), P(self.k_eff_tiles), P(self.ckpt_mask), P(self.work),
                self.work_capacity, P(self.status), n, P(buf), stream_handle()),
                "ss_contributed_from_masks")
            self.contributed_buf = buf[:n].view(torch.bool)
        return self.contributed_buf

    @property
    def acc_rgb(self) -> torch.Tensor:
        bg = torch.tensor(self.opts.background, dtype=torch.float32, device=self.image.device)
        return self.image - bg * self.final_t[..., None]

    @property
    def alpha(self) -> torch.Tensor:
        """Builder extension A15: 1 - final_T (kernels.py:102)."""
        return 1.0 - self.final_t

    @property
    def checkpoints(self):
        return None if self.ckpt is None else self.ckpt

    @property
    def proj(self) -> Projection:
        if "proj" not in self._cache:
            p = _projection_from_splats(self.splats, self.opts.sh_degree)
            p._device = (self.splats, self.camera, self.gmap, self.opts)
            self._cache["proj"] = p
        return self._cache["proj"]

    @property
    def tile_index(self) -> TileIndex:
        if "ti" not in self._cache:
            W, H = self.camera.width, self.camera.height
            tx, ty = (W + 15) // 16, (H + 15) // 16
            pg = self.bins.pairs[:self.pair_count].cpu().numpy().astype(np.int64)
            st = self.bins.tile_start.cpu().numpy().astype(np.int64)
            en = self.bins.tile_end.cpu().numpy().astype(np.int64)
            ln = en - st
            rng = np.zeros(tx * ty + 1, dtype=np.int64)
            np.cumsum(ln, out=rng[1:])
            row = np.full(self.n_primitives, -1, dtype=np.int64)
            row[self.proj.map_index] = np.arange(len(self.proj))
            self._cache["ti"] = TileIndex(16, tx, ty, row[pg].astype(np.int32), pg, rng,
                                          np.flatnonzero(ln > 0).astype(np.int64))
        return self._cache["ti"]

    @property
    def k_eff(self) -> np.ndarray:
        """Per active tile, in active-tile order (api.py:195)."""
        ke = self.k_eff_tiles.cpu().numpy().astype(np.int64)
        return ke[self.tile_index.active_tiles]


def _as_image(x, shape, dev, name="grad_image"):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    x = x.to(device=dev, dtype=torch.float32).contiguous()
    return x


def _bin(sp: SplatBuffers, n: int, cam: Camera, dev, st):
    """K2-K4b with pair-capacity retry: (BinBuffers, pair count, status +
    checkpoint-slot total as one host read)."""
    L = lib()
    s = stream_handle()
    tx, ty = cam.tiles
    n_tiles = tx * ty
    cm = cam.to_ss()
    key = (str(dev), n_tiles)
    cap = max(_CAP_HINT.get(key, 0), 4 * n, 1024)
    while True:
        bins = BinBuffers.alloc(cap, n_tiles, dev)
        cost = _COST_HINT.get(key)
        if cost is None:
            cost = _COST_HINT[key] = bins.tile_cost
        bins.tile_cost = cost
        ws = bin_workspace(n, cap, n_tiles, dev)
        check(L.ss_bin_sort(n, ctypes.byref(sp.ss()), ctypes.byref(cm), ctypes.byref(bins.ss()),
                            P(ws), ws.numel(), P(st), s), "ss_bin_sort")
        # status words + the checkpoint slot total in one host read (with every
        # check a deferred-error call left pending, errors.py)
        sh = errors.read_with_pending(
            torch.cat((st, bins.ckpt_base[n_tiles:n_tiles + 1].to(torch.int64))))
        raise_param_errors(sh[:-1])
        pcount = int(sh[_lib.ST_PAIRS])
        if not int(sh[_lib.ST_OVERFLOW]):
            break
        st[_lib.ST_OVERFLOW] = 0  # the overflow word is sticky; clear it for the retry
        cap = int(pcount * 1.25) + 1024
    _CAP_HINT[key] = cap
    return bins, pcount, sh


@traced("ss.project_map")
def project_map(gmap: GaussianMap, camera, *, dtype=np.float32, sh_degree: int = 3,
                near: float = 0.01, dilation: float = 0.3,
                alpha_min: float = 1.0 / 255.0) -> Projection:
    """projection.py:73-163 as K1 on the GPU: every primitive projected,
    splats behind the near plane or missing the image culled; returns the
    reference-shaped (compacted) Projection.  The B200 path computes in
    float32 (``dtype`` only sets the returned arrays' type); the backward
    context fields (cov_cam, rot, q_hat, ...) are not materialised: the
    chain recomputes them from the map (chain_backward below)."""
    cam = Camera.of(camera)
    opts = RasterOpts(sh_degree=sh_degree, near=near, dilation=dilation, alpha_min=alpha_min)
    dev = gmap.device
    st = new_status(dev)
    sp = SplatBuffers.alloc(len(gmap), dev)
    mp, cm, op = gmap.ss(), cam.to_ss(), opts.to_ss()
    check(lib().ss_preprocess(ctypes.byref(mp), ctypes.byref(cm), None, ctypes.byref(op),
                              ctypes.byref(sp.ss()), P(st), stream_handle()), "ss_preprocess")
    raise_param_errors(st.cpu())
    p = _projection_from_splats(sp, sh_degree, dtype)
    p._device = (sp, cam, gmap, opts)
    return p


@traced("ss.build_tile_index")
def build_tile_index(proj: Projection, width: int, height: int, tile_size: int = 16) -> TileIndex:
    """tiles.py:29-65 on the GPU (K2-K4b): inclusive tile rects, pairs sorted
    by (tile, depth, row), tile ranges and active tiles -- bit-exact with the
    reference on a float32 projection.  A Projection from project_map (or
    RenderOutput.proj) is binned from its device buffers; any other
    reference-shaped projection (numpy mean2d / radius / depth) is uploaded
    as float32 first (ss_splats_from_projection)."""
    if tile_size != 16:
        raise ValueError("the B200 kernels are specialised for tile_size=16")
    W, H = int(width), int(height)
    dv = getattr(proj, "_device", None)
    if dv is not None and (dv[1].width, dv[1].height) == (W, H):
        sp, cam = dv[0], dv[1]
        n = int(sp.flags.numel())
        dev = sp.flags.device
        st = new_status(dev)
        bins, pcount, _ = _bin(sp, n, cam, dev, st)
        pg = bins.pairs[:pcount].cpu().numpy().astype(np.int64)
        row = np.full(n, -1, dtype=np.int64)
        row[proj.map_index] = np.arange(len(proj))
        rows = row[pg]
    else:
        dev = torch.device("cuda")
        m = len(proj)
        cam = Camera(1.0, 1.0, W / 2.0, H / 2.0, W, H)  # only the image size is used
        sp = SplatBuffers.alloc(m, dev, aux=False)
        f32 = (lambda a, shp: torch.as_tensor(np.ascontiguousarray(a, np.float32).reshape(shp))
               .to(dev))
        mean2d, radius, depth = f32(proj.mean2d, (m, 2)), f32(proj.radius, (m,)), f32(proj.depth,
                                                                                    (m,))
        check(lib().ss_splats_from_projection(m, P(mean2d), P(radius), P(depth),
                                              ctypes.byref(cam.to_ss()), ctypes.byref(sp.ss()),
                                              stream_handle()), "ss_splats_from_projection")
        st = new_status(dev)
        bins, pcount, _ = _bin(sp, m, cam, dev, st)
        rows = bins.pairs[:pcount].cpu().numpy().astype(np.int64)
        pg = rows
    tx, ty = cam.tiles
    st_ = bins.tile_start.cpu().numpy().astype(np.int64)
    en = bins.tile_end.cpu().numpy().astype(np.int64)
    ln = en - st_
    rng = np.zeros(tx * ty + 1, dtype=np.int64)
    np.cumsum(ln, out=rng[1:])
    return TileIndex(16, tx, ty, rows.astype(np.int32), pg, rng,
                     np.flatnonzero(ln > 0).astype(np.int64))


@traced("ss.chain_backward")
def chain_backward(proj: Projection, camera, g2d, n_primitives: int) -> dict:
    """projection.py:200-299 as K8 on the GPU: per-splat screen-space rows
    g2d (M, 9) [rgb3, mean2d2, conic3, opacity] -> dense float32 device
    gradients over the map (culled primitives get zeros) plus the
    pos2d_grad_norm densify statistic.  The projection context is
    recomputed from the map's parameters, so ``proj`` must come from
    project_map / RenderOutput.proj."""
    if getattr(proj, "_device", None) is None:
        raise ValueError("chain_backward on the B200 path needs a Projection from project_map "
                         "(the chain recomputes the projection context from the map)")
    sp, pcam, gmap, opts = proj._device
    cam = Camera.of(camera)
    n = int(n_primitives)
    if n != len(gmap):
        raise ValueError(f"n_primitives {n} does not match the projected map ({len(gmap)})")
    dev = gmap.device
    rows = torch.as_tensor(np.asarray(g2d, np.float32) if not isinstance(g2d, torch.Tensor)
                           else g2d, dtype=torch.float32).to(dev).reshape(len(proj), -1)
    full = torch.zeros((max(n, 1), 9), dtype=torch.float32, device=dev)
    if len(proj):
        full[torch.as_tensor(proj.map_index.astype(np.int64), device=dev)] = rows[:, :9]
    grads = ParamGrads.alloc(n, dev)
    st = new_status(dev)
    mp, cm, op = gmap.ss(), cam.to_ss(), opts.to_ss()
    check(lib().ss_chain_backward(ctypes.byref(mp), ctypes.byref(cm), ctypes.byref(op), P(full),
                                  P(sp.flags), None, 0.0, 0, ctypes.byref(grads.ss()), P(st),
                                  stream_handle()), "ss_chain_backward")
    return {"position": grads.position, "rotation": grads.rotation,
            "log_scale": grads.log_scale, "opacity_logit": grads.opacity_logit,
            "sh": grads.sh, "pos2d_grad_norm": grads.pos2d_grad_norm}


@traced("ss.replay_pixel_states")
def replay_pixel_states(render: "RenderOutput", tile_pos: int, from_bucket: int,
                        n_positions: int | None = None):
    """api.py:340-368: advance the archived pixel states of active tile
    ``tile_pos`` from checkpoint bucket ``from_bucket`` by ``n_positions``
    list positions (default: to the tile's processed prefix k_eff).  Returns
    host float32 arrays (T (npx,), rgb (npx, 3)) over the tile's pixels,
    row-major; a replay to k_eff reproduces the forward's final states bit
    for bit."""
    if render.ckpt is None:
        raise RuntimeError("render output has no checkpoints")
    ti = render.tile_index
    tile = int(ti.active_tiles[tile_pos])
    ke = int(render.k_eff[tile_pos])
    nb = (ke + 31) // 32
    if not 0 <= from_bucket < nb:
        raise IndexError(f"bucket {from_bucket} out of range for a tile with {nb} checkpoints")
    pos_from = from_bucket * 32
    pos_to = ke if n_positions is None else min(ke, pos_from + int(n_positions))
    x0, y0 = ti.tile_origin(tile)
    tw = min(16, render.camera.width - x0)
    th = min(16, render.camera.height - y0)
    out = torch.empty((th * tw, 4), dtype=torch.float32, device=render.image.device)
    cm, op = render.camera.to_ss(), render.opts.to_ss()
    check(lib().ss_replay_pixel_states(ctypes.byref(cm), ctypes.byref(op),
                                       ctypes.byref(render.splats.ss()),
                                       ctypes.byref(render.bins.ss()), P(render.image),
                                       P(render.final_t), P(render.n_contrib), P(render.ckpt),
                                       tile, int(from_bucket), int(pos_to), P(out),
                                       stream_handle()), "ss_replay_pixel_states")
    h = out.cpu().numpy()
    return h[:, 0].copy(), h[:, 1:4].copy()


@traced("ss.rasterize_forward")
def rasterize_forward(gmap: GaussianMap, camera, opts: RasterOpts | None = None) -> RenderOutput:
    """api.py:118-206 on the GPU: K1 preprocess -> K2-K4b binning -> K5 blend."""
    if opts is None:
        opts = RasterOpts()
    cam = Camera.of(camera)
    L = lib()
    dev = gmap.device
    n = len(gmap)
    H, W = cam.height, cam.width
    tx, ty = cam.tiles
    n_tiles = tx * ty
    s = stream_handle()
    st = new_status(dev)
    sp = SplatBuffers.alloc(n, dev)
    mp, cm, op = gmap.ss(), cam.to_ss(), opts.to_ss()
    check(L.ss_preprocess(ctypes.byref(mp), ctypes.byref(cm), None, ctypes.byref(op),
                          ctypes.byref(sp.ss()), P(st), s), "ss_preprocess")
    bins, pcount, sh = _bin(sp, n, cam, dev, st)
    n_slots = int(sh[-1])
    f32 = dict(dtype=torch.float32, device=dev)
    ckpt = torch.empty((max(n_slots, 1) * 256, 4), **f32)
    ckpt_depth = torch.empty(max(n_slots, 1) * 256, **f32) if opts.with_depth else None
    ckpt_mask = torch.empty(max(n_slots, 1) * 256, dtype=torch.int32, device=dev)
    image = torch.empty((H, W, 3), **f32)
    final_t = torch.empty((H, W), **f32)
    n_contrib = torch.empty((H, W), dtype=torch.int32, device=dev)
    depth = torch.empty((H, W), **f32) if opts.with_depth else None
    k_eff = torch.empty(n_tiles, dtype=torch.int32, device=dev)
    work_cap = max(n_slots, 1)
    work = torch.empty((work_cap, 2), dtype=torch.int32, device=dev)
    check(L.ss_blend_forward(ctypes.byref(cm), ctypes.byref(op), ctypes.byref(sp.ss()),
                             ctypes.byref(bins.ss()), P(image), P(final_t), P(n_contrib), P(depth),
                             P(k_eff), None, P(ckpt), P(ckpt_depth), P(ckpt_mask),
                             P(work), work_cap, P(st), s), "ss_blend_forward")
    return RenderOutput(image=image, final_t=final_t, n_contrib=n_contrib, k_eff_tiles=k_eff,
                        contributed_buf=None, opts=opts, camera=cam, n_primitives=n,
                        gmap=gmap, splats=sp, bins=bins, pair_count=pcount,
                        ckpt=ckpt if opts.with_checkpoints else None, ckpt_depth=ckpt_depth,
                        ckpt_mask=ckpt_mask, work=work, work_capacity=work_cap, status=st, depth=depth)


@dataclass
class ParamGrads:
    """api.py:55-79, float32 device tensors; ``sh`` is assembled on request."""

    position: torch.Tensor
    rotation: torch.Tensor
    log_scale: torch.Tensor
    opacity_logit: torch.Tensor
    sh_dc: torch.Tensor
    sh_rest: torch.Tensor
    pos2d_grad_norm: torch.Tensor
    contributed: torch.Tensor
    sh_degree: int | None = None  # of the render they came from (None: unknown)
    # tensors an eager check found finite: name -> (id, torch version, any
    # non-zero); adam_step re-checks only tensors replaced or modified since
    _finite_ok: dict = field(default_factory=dict, repr=False, compare=False)

    def __len__(self):
        return int(self.position.shape[0])

    @property
    def sh(self) -> torch.Tensor:
        n = len(self)
        return torch.cat([self.sh_dc.view(n, 1, 3), self.sh_rest.view(n, 15, 3)], 1)

    @classmethod
    def alloc(cls, n, dev, zero=False):
        mk = torch.zeros if zero else torch.empty
        f = dict(dtype=torch.float32, device=dev)
        return cls(mk((n, 3), **f), mk((n, 4), **f), mk((n, 3), **f), mk(n, **f), mk((n, 3), **f),
                   torch.zeros((n, 45), **f), mk(n, **f), torch.zeros(n, dtype=torch.bool,
                                                                     device=dev))

    def ss(self):
        g = _lib.SSParamGrads()
        g.d_position, g.d_rotation, g.d_log_scale = P(self.position), P(self.rotation), P(
            self.log_scale)
        g.d_opacity, g.d_sh_dc, g.d_sh_rest = P(self.opacity_logit), P(self.sh_dc), P(self.sh_rest)
        g.d_pos2d_norm = P(self.pos2d_grad_norm)
        return g

    def validate_finite(self):
        """api.py:74-79 (one fused reduction, one host read; in deferred error
        mode the check stays on the device and raises later, errors.py)."""
        names = ("position", "rotation", "log_scale", "opacity_logit", "sh_dc", "sh_rest")

        def raiser(bad):
            for k, b in zip(names, [int(v) for v in bad[:len(names)]]):
                if b:
                    raise FloatingPointError(
                        f"non-finite gradient in {'sh' if k.startswith('sh') else k}")
        tensors = [getattr(self, k) for k in names]
        if errors.deferred():
            errors.defer(finite_flags_device(tensors)[:len(names)], raiser)
        else:
            host = finite_flags(tensors, extra_nonzero=True)
            raiser([0 if good else 1 for good in host[:len(names)]])
            self.note_finite(names, tensors, host[len(names):])
        return self

    def note_finite(self, names, tensors, nonzero):
        for k, t, nz in zip(names, tensors, nonzero):
            self._finite_ok[k] = (id(t), t._version, bool(nz))

    def known_finite(self, name, t):
        """(known finite, any non-zero) for tensor `t` held as `name`: a
        tensor an eager check passed and nothing has modified in place since
        (torch version counter) needs no second reduction."""
        rec = self._finite_ok.get(name)
        if rec is not None and rec[0] == id(t) and rec[1] == t._version:
            return True, rec[2]
        return False, None


def render_trajectory(gmap: GaussianMap, cameras, opts: RasterOpts | None = None):
    """trainer.py:271-279: one image per camera, forward only (no checkpoints)."""
    opts = opts if opts is not None else RasterOpts()
    opts = dataclasses.replace(opts, with_checkpoints=False)
    return [rasterize_forward(gmap, cam, opts).image for cam in cameras]


def screen_space_grads(render: RenderOutput, grad_image, grad_depth=None):
    """K7 only: the per-Gaussian screen-space rows g2d (N, 9|10) float32 the
    reference merges before chain_backward (api.py:331-336)."""
    if render.ckpt is None:
        raise RuntimeError("render output has no checkpoints; re-run rasterize_forward "
                           "with with_checkpoints=True to use the splat-wise backward")
    dev = render.image.device
    if tuple(grad_image.shape) != tuple(render.image.shape):
        raise ValueError(f"grad_image shape {tuple(grad_image.shape)} does not match "
                         f"rendered image shape {tuple(render.image.shape)}")
    g = _as_image(grad_image, render.image.shape, dev)
    gd = None
    if render.opts.with_depth:
        gd = (_as_image(grad_depth, render.depth.shape, dev) if grad_depth is not None
              else torch.zeros_like(render.depth))
    ncol = 10 if render.opts.with_depth else 9
    n = render.n_primitives
    g2d = torch.empty((max(n, 1), ncol), dtype=torch.float32, device=dev)
    cm, op = render.camera.to_ss(), render.opts.to_ss()
    check(lib().ss_backward_schedule(ctypes.byref(cm), P(render.k_eff_tiles), P(render.work),
                                     render.work_capacity, P(render.status), stream_handle()),
          "ss_backward_schedule")
    check(lib().ss_backward_splat(
        ctypes.byref(cm), ctypes.byref(op), ctypes.byref(render.splats.ss()),
        ctypes.byref(render.bins.ss()), P(render.image), P(g), None, P(render.depth), P(gd),
        P(render.n_contrib), P(render.k_eff_tiles), P(render.ckpt), P(render.ckpt_depth),
        P(render.ckpt_mask), P(render.work), render.work_capacity, n, P(g2d), None,
        P(render.status),
        stream_handle()), "ss_backward_splat")
    return g2d[:n]


@traced("ss.backward_splatwise")
def backward_splatwise(render: RenderOutput, grad_image, n_workers=None,
                       grad_depth=None) -> ParamGrads:
    """api.py:275-337: K7 splat-wise backward + K8 chain to parameters."""
    g2d = screen_space_grads(render, grad_image, grad_depth)
    return _finish_backward(render, g2d)


def screen_space_grads_pixelwise(render: RenderOutput, grad_image):
    """F2 (api.py:227-272): the pixel-parallel backward up to the screen-space
    rows g2d (N, 9), the paper's ablation baseline for the splat-wise K7."""
    if render.opts.with_depth:
        raise ValueError("backward_pixelwise does not support the depth extension")
    dev = render.image.device
    if tuple(grad_image.shape) != tuple(render.image.shape):
        raise ValueError(f"grad_image shape {tuple(grad_image.shape)} does not match "
                         f"rendered image shape {tuple(render.image.shape)}")
    g = _as_image(grad_image, render.image.shape, dev)
    n = render.n_primitives
    g2d = torch.empty((max(n, 1), 9), dtype=torch.float32, device=dev)
    cm, op = render.camera.to_ss(), render.opts.to_ss()
    check(lib().ss_backward_pixel(
        ctypes.byref(cm), ctypes.byref(op), ctypes.byref(render.splats.ss()),
        ctypes.byref(render.bins.ss()), P(render.image), P(g), P(render.n_contrib),
        P(render.k_eff_tiles), n, P(g2d), stream_handle()), "ss_backward_pixel")
    return g2d[:n]


@traced("ss.backward_pixelwise")
def backward_pixelwise(render: RenderOutput, grad_image, n_workers=None) -> ParamGrads:
    """api.py:227-272: pixel-parallel backward + K8 chain to parameters (the
    reference's alternative to backward_splatwise; no checkpoints needed)."""
    g2d = screen_space_grads_pixelwise(render, grad_image)
    return _finish_backward(render, g2d)


def _finish_backward(render: RenderOutput, g2d) -> ParamGrads:
    """api.py:217-224: chain_backward + validate_finite."""
    n = render.n_primitives
    dev = render.image.device
    grads = ParamGrads.alloc(n, dev)
    grads.contributed = render.contributed.clone()
    grads.sh_degree = render.opts.sh_degree
    mp, cm, op = render.gmap.ss(), render.camera.to_ss(), render.opts.to_ss()
    check(lib().ss_chain_backward(ctypes.byref(mp), ctypes.byref(cm), ctypes.byref(op), P(g2d),
                                  P(render.splats.flags), None, 0.0, 0, ctypes.byref(grads.ss()),
                                  P(render.status), stream_handle()), "ss_chain_backward")
    return grads.validate_finite()
