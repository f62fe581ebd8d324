"""The mapping iteration as one stream-ordered sequence of B200 kernels.

``MappingEngine.step`` is ``_Trainer.train_one`` (trainer.py:180-215) for
one keyframe view, without host synchronisation:

  K1 preprocess -> K2-K4b binning -> K5 blend -> K6 L1+SSIM (+depth) ->
  K7 splat-wise backward -> K8+K9 fused chain + opacity-reg grad + stats +
  Adam (one kernel; the per-Gaussian gradients never reach HBM)

All buffers are allocated once for the map size, image size and pair
capacity.  Data-dependent sizes stay on the device: the pair count P only
has to fit the capacity; if it does not, the binning sets a sticky
overflow word, the fused update becomes a no-op, and the host -- which
reads each step's status block two steps late through pinned memory --
grows the buffers and replays the skipped steps in order.  The loss
scalars are read the same way (``losses()``), so the scheduler-style
consumer never stalls the GPU.

``multiview_step`` is the builder-defined keyframe batch (SURVEY 8a A17,
8e): per-view K1-K7 + accumulate-mode K8 into one flat gradient buffer
(grads + densify-statistics increments), an optional all-reduce hook
(torch.distributed / NCCL over NVLink), then K9 Adam and the statistics
update -- identical on every rank.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import SS_BWD_SKIP_CLEAR, check, lib, traced
from .core import Camera, GaussianMap
from .densify import DensifyConfig, densify_and_prune, opacity_reset
from .optimizer import AdamState, LearningRates
from .rasterizer import BinBuffers, P, RasterOpts, SplatBuffers, bin_workspace, stream_handle

STATUS_LAG = 2

# kernels each C-ABI call enqueues (counted for bench.py's gpu_launches)
KERNELS_PER_CALL = {
    # status_begin 1 + preprocess 1 + blend 1 + loss (ssim fwd, ssim bwd with
    # the partial-sum reduction) 2 + backward (clear, schedule, splat-wise) 3;
    # binning is counted separately (binning_kernels)
    "step_fb": 1 + 1 + 1 + 2 + 3,
    "chain_adam": 1,
    "snapshot": 1,
    "tile_order": 1,  # ss_tile_order on the side stream
}


def binning_kernels(n_tiles: int, n: int = 0) -> int:
    """Kernels of one ss_bin_sort (binning.cu) as the engine calls it (no
    tile order: that is ss_tile_order on the side stream).  Up to ~1.2M
    splats the front end is one cooperative kernel; with <= 8192 tiles it also
    places the pairs and writes the checkpoint bases (clear + front end),
    else clear + front end + tile passes x 3 + ranges + checkpoint-base scan;
    beyond ~1.2M splats the front end is 4 x 3 radix kernels + scan + emit +
    clamp."""
    bits = max(1, (n_tiles - 1).bit_length())
    if n <= 148 * 8192 and n_tiles <= 8192:
        return 1 + 1
    front = 1 if n <= 148 * 8192 else 4 * 3 + 1 + 1 + 1
    return 1 + front + 3 * ((bits + 7) // 8) + 1 + 1


@dataclass
class StepRecord:
    index: int
    camera: Camera
    target: torch.Tensor
    target_depth: torch.Tensor | None
    hp: _lib.SSAdamHP
    slot: int
    event: torch.cuda.Event
    replayed: int = 0


@dataclass
class EngineConfig:
    lambda_ssim: float = 0.2
    lambda_o: float = 0.001
    depth_weight: float = 0.0          # builder extension A15 (RGB-D configs)
    densify: DensifyConfig | None = None
    scene_extent: float = 1.0
    opacity_reset_interval: int = 0    # builder extension A16 (0 = off)
    opacity_reset_ceiling: float = 0.01
    pair_margin: float = 1.3
    lrs: LearningRates = field(default_factory=LearningRates)
    horizon: int = 30000


class MappingEngine:
    """Owns the device buffers of the fused mapping iteration for one map."""

    def __init__(self, gmap: GaussianMap, width: int, height: int, opts: RasterOpts | None = None,
                 config: EngineConfig | None = None, pair_capacity: int | None = None):
        self.gmap = gmap
        self.opts = opts or RasterOpts(sh_degree=0)
        self.cfg = config or EngineConfig()
        self.W, self.H = int(width), int(height)
        self.dev = gmap.device
        self.state = AdamState.for_map(gmap, self.cfg.lrs, self.cfg.horizon)
        self.tiles_x, self.tiles_y = (self.W + 15) // 16, (self.H + 15) // 16
        self.n_tiles = self.tiles_x * self.tiles_y
        self.iteration = 0
        self.since_densify = 0
        self._records: list[StepRecord] = []
        self._loss_log: list[tuple[int, float, float]] = []
        self._cap = int(pair_capacity) if pair_capacity else max(16 * len(gmap), 4096)
        self.status = torch.empty(_lib.STATUS_WORDS, dtype=torch.int64, device=self.dev)
        check(lib().ss_status_reset(P(self.status), stream_handle()), "ss_status_reset")
        self._slots = 8
        # page-locked snapshot rows written by ss_step_snapshot (one kernel)
        self._host = torch.zeros((self._slots, _lib.SNAPSHOT_DOUBLES), dtype=torch.float64,
                                 pin_memory=True)
        self._graphs: dict = {}
        self._cam_last = None  # (caller's camera, its key, Camera, ss_camera)
        self._alloc_map_buffers()
        self._alloc_pair_buffers(self._cap)
        self.profile = None  # list of (stage, start event, end event) when profiling
        self.launches = 0    # kernels launched by this engine (see KERNELS_PER_CALL)
        # per-step parameters (camera, Adam step values) live in device memory
        # so one captured CUDA graph serves every step; they are filled from a
        # ring of pinned host slots (a slot is reused only after its step drained)
        self._pslots = 8
        self._pbytes = 256
        self._phost = torch.zeros((self._pslots, self._pbytes), dtype=torch.uint8,
                                  pin_memory=True)
        self._pdev = torch.zeros(self._pbytes, dtype=torch.uint8, device=self.dev)
        self.use_graph = False
        self._mv_unchecked = False

    def enable_graph(self, on: bool = True):
        """Replay the iteration body from ONE captured CUDA graph (the step's
        target is copied into target_buffer(), the camera and Adam values
        into a device parameter block); buffers reallocated by densify or
        capacity growth drop the capture."""
        self.use_graph = on
        self._graphs.clear()

    def _params_ptrs(self):
        base = self._pdev.data_ptr()
        return ctypes.c_void_p(base), ctypes.c_void_p(base + 128)

    def _slot_event(self, it):
        """The snapshot event of slot it % slots (created once: a slot's
        record is drained long before the slot comes round again)."""
        if getattr(self, "_events", None) is None:
            self._events = [None] * self._slots
        k = it % self._slots
        if self._events[k] is None:
            self._events[k] = torch.cuda.Event()
        return self._events[k]

    def _camera_of(self, camera):
        """Camera.of(camera) and its ss_camera struct, reused while the caller
        passes the same, unchanged camera object (host time before the step's
        first launch: the GPU waits for it)."""
        key = (camera.fx, camera.fy, camera.cx, camera.cy, int(camera.width),
               int(camera.height), np.asarray(camera.R).tobytes(), np.asarray(camera.t).tobytes())
        c = self._cam_last
        if c is not None and c[0] is camera and c[1] == key:
            return c[2]
        cam = Camera.of(camera)
        self._cam_last = (camera, key, cam, cam.to_ss())
        return cam

    def _stage_params(self, rec):
        """Write the step's camera + Adam values into its pinned slot and
        enqueue the host->device copy."""
        slot = self._phost[rec.slot % self._pslots]
        c = self._cam_last
        cm = c[3] if c is not None and c[2] is rec.camera else rec.camera.to_ss()
        ctypes.memmove(slot.data_ptr(), ctypes.addressof(cm), ctypes.sizeof(cm))
        ctypes.memmove(slot.data_ptr() + 128, ctypes.addressof(rec.hp), ctypes.sizeof(rec.hp))
        self._pdev.copy_(slot, non_blocking=True)

    def _mark(self, name):
        """Stage boundary: an NVTX marker (profiler timelines) and, when
        profiling, an event for the per-kernel timing bench.py reports."""
        torch.cuda.nvtx.mark("ss." + name)
        if self.profile is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.profile.append((name, ev))

    # ------------------------------------------------------------ buffers
    def _alloc_map_buffers(self):
        self._graphs.clear()
        n = len(self.gmap)
        dev = self.dev
        self.splats = self.g2d = self.contributed = None  # blocks reusable below
        self.splats = SplatBuffers.alloc(n, dev, aux=False)
        ncol = 10 if self.opts.with_depth else 9
        self.g2d = torch.empty((max(n, 1), ncol), dtype=torch.float32, device=dev)
        self.contributed = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
        self._flat = None
        if getattr(self, "image", None) is not None:
            return  # the image-sized buffers do not depend on the map size
        f32 = dict(dtype=torch.float32, device=dev)
        self.image = torch.empty((self.H, self.W, 3), **f32)
        self.final_t = torch.empty((self.H, self.W), **f32)
        self.n_contrib = torch.empty((self.H, self.W), dtype=torch.int32, device=dev)
        self.depth = torch.empty((self.H, self.W), **f32) if self.opts.with_depth else None
        self.grad_depth = torch.empty((self.H, self.W), **f32) if self.opts.with_depth else None
        self.grad_image = torch.empty((self.H, self.W, 3), **f32)
        self.pixgrad = torch.empty((self.H, self.W, 4), **f32)
        self.k_eff = torch.empty(self.n_tiles, dtype=torch.int32, device=dev)
        self.sums = torch.zeros(_lib.SS_REDUCE_DOUBLES, dtype=torch.float64, device=dev)
        self.dsum = torch.zeros(_lib.SS_REDUCE_DOUBLES, dtype=torch.float64, device=dev)
        self.loss_ws = torch.empty(int(lib().ss_loss_workspace_bytes(self.H, self.W)),
                                   dtype=torch.uint8, device=dev)
        if getattr(self, "_tgt_buf", None) is None:
            self._tgt_buf = torch.zeros((self.H, self.W, 3), **f32)
            self._tgt_buf1 = None
            self._tdep_buf = None
        self._flat = None

    def _alloc_pair_buffers(self, cap):
        self._graphs.clear()
        n = len(self.gmap)
        self._cap = int(cap)
        # drop the old buffers first so the caching allocator can hand their
        # blocks to the new ones
        self.bins = self.bin_ws = self.ckpt = self.ckpt_depth = self.ckpt_mask = None
        self.work = None
        self.bins = BinBuffers.alloc(self._cap, self.n_tiles, self.dev)
        self.bin_ws = bin_workspace(n, self._cap, self.n_tiles, self.dev)
        slots = self._cap // 32 + self.n_tiles + 1
        self.ckpt = torch.empty((slots * 256, 4), dtype=torch.float32, device=self.dev)
        self.ckpt_depth = (torch.empty(slots * 256, dtype=torch.float32, device=self.dev)
                           if self.opts.with_depth else None)
        self.ckpt_mask = torch.empty(slots * 256, dtype=torch.int32, device=self.dev)
        self.work_cap = slots
        self.work = torch.empty((slots, 2), dtype=torch.int32, device=self.dev)

    @property
    def pair_capacity(self):
        return self._cap

    # -------------------------------------------------------------- pieces
    def _forward_backward(self, cam: Camera, target: torch.Tensor, target_depth, view_mode):
        """K1..K7 for one view; view_mode None = fused single view."""
        L = lib()
        s = stream_handle()
        mp, cm, op = self.gmap.ss(), cam.to_ss(), self.opts.to_ss()
        spss, bss = self.splats.ss(), self.bins.ss()
        n = len(self.gmap)
        self._mark("begin")
        # the forward's tile order (costliest first, from the last forward's
        # per-tile costs) on a side stream, overlapping the projection; joined
        # before the cooperative binning launch, which then leaves the order
        # alone (its ss_bins copy has no cost array)
        side = self._side_stream()
        bss_sort = bss
        if bss.d_tile_order and bss.d_tile_cost:
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                check(L.ss_tile_order(ctypes.byref(cm), ctypes.byref(bss), stream_handle()),
                      "ss_tile_order")
            bss_sort = self.bins.ss()
            bss_sort.d_tile_cost = None
        check(L.ss_status_begin_step(P(self.status), s), "ss_status_begin_step")
        d_cam = self._params_ptrs()[0] if view_mode is None else None
        check(L.ss_preprocess(ctypes.byref(mp), ctypes.byref(cm), d_cam, ctypes.byref(op),
                              ctypes.byref(spss), P(self.status), s), "ss_preprocess")
        self._mark("preprocess")
        torch.cuda.current_stream().wait_stream(side)
        check(L.ss_bin_sort(n, ctypes.byref(spss), ctypes.byref(cm), ctypes.byref(bss_sort),
                            P(self.bin_ws), self.bin_ws.numel(), P(self.status), s),
              "ss_bin_sort")
        self._mark("binning")
        check(L.ss_blend_forward(ctypes.byref(cm), ctypes.byref(op), ctypes.byref(spss),
                                 ctypes.byref(bss), P(self.image), P(self.final_t),
                                 P(self.n_contrib), P(self.depth), P(self.k_eff), None,
                                 P(self.ckpt), P(self.ckpt_depth), P(self.ckpt_mask),
                                 P(self.work), self.work_cap, P(self.status), s),
              "ss_blend_forward")
        self._mark("blend_forward")
        # the backward's longest-units-first schedule (needs only k_eff): on a
        # side stream, concurrent with the loss kernels (fork / join by events,
        # captured into the step's graph like the main stream)
        side = self._side_stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            check(L.ss_backward_schedule(ctypes.byref(cm), P(self.k_eff), P(self.work),
                                         self.work_cap, P(self.status), stream_handle()),
                  "ss_backward_schedule")
            # the backward's clearing of the g2d rows (last read by the
            # previous step's chain+Adam) off the critical path as well
            check(L.ss_backward_clear(n, 10 if self.opts.with_depth else 9, P(self.g2d),
                                      P(self.contributed), P(self.status), stream_handle()),
                  "ss_backward_clear")
        use_pg = self.cfg.lambda_ssim != 0.0 and not self.opts.with_depth
        # with pixgrad the backward never reads grad_image: it is not written
        check(L.ss_loss_l1_ssim(self.H, self.W, P(self.image), P(target),
                                float(self.cfg.lambda_ssim),
                                None if use_pg else P(self.grad_image),
                                P(self.pixgrad) if use_pg else None, P(self.sums),
                                P(self.loss_ws), self.loss_ws.numel(), s), "ss_loss_l1_ssim")
        if self.opts.with_depth:
            if target_depth is not None and self.cfg.depth_weight != 0.0:
                check(L.ss_depth_l1(self.H, self.W, P(self.depth), P(target_depth),
                                    float(self.cfg.depth_weight), P(self.grad_depth),
                                    P(self.dsum), s), "ss_depth_l1")
            else:
                self.grad_depth.zero_()
        self._mark("loss")
        torch.cuda.current_stream().wait_stream(side)
        check(L.ss_backward_splat_ex(ctypes.byref(cm), ctypes.byref(op), ctypes.byref(spss),
                                     ctypes.byref(bss), P(self.image), P(self.grad_image),
                                     P(self.pixgrad) if use_pg else None, P(self.depth),
                                     P(self.grad_depth), P(self.n_contrib), P(self.k_eff),
                                     P(self.ckpt), P(self.ckpt_depth), P(self.ckpt_mask),
                                     P(self.work), self.work_cap, n, P(self.g2d),
                                     P(self.contributed), P(self.status), SS_BWD_SKIP_CLEAR, s),
              "ss_backward_splat_ex")
        self._mark("backward")
        return mp, cm, op

    def _side_stream(self):
        if getattr(self, "_side", None) is None or self._side.device != self.dev:
            self._side = torch.cuda.Stream(device=self.dev)
        return self._side

    def _snapshot(self, rec: StepRecord):
        """Copy the step's status block + loss sums into its pinned slot."""
        row = self._host[rec.slot]
        check(lib().ss_step_snapshot(P(self.status), P(self.sums), row.data_ptr(),
                                     stream_handle()), "ss_step_snapshot")
        rec.event.record()

    # ---------------------------------------------------------- main step
    @traced("ss.MappingEngine.step")
    def step(self, camera, target: torch.Tensor, target_depth: torch.Tensor | None = None):
        """One fused mapping iteration (single view, single GPU)."""
        self._maybe_densify()
        cam = self._camera_of(camera)
        self.state.step_count += 1
        hp = self.state.hparams(self.opts.sh_degree > 0)
        rec = StepRecord(self.iteration, cam, target, target_depth, hp,
                         self.iteration % self._slots, self._slot_event(self.iteration))
        self._run(rec)
        self._records.append(rec)
        self.iteration += 1
        self.since_densify += 1
        self._drain(STATUS_LAG)
        return rec.index

    def _body(self, cam: Camera, target, target_depth):
        """The iteration's kernels; the per-step camera / Adam values are read
        from the device parameter block (graph-capturable)."""
        L = lib()
        n = len(self.gmap)
        mp, cm, op = self._forward_backward(cam, target, target_depth, None)
        lon = float(self.cfg.lambda_o / n) if n else 0.0
        d_cam, d_hp = self._params_ptrs()
        hp0 = self.state.hparams(self.opts.sh_degree > 0)
        check(L.ss_chain_adam(ctypes.byref(mp), ctypes.byref(cm), d_cam, ctypes.byref(op),
                              P(self.g2d), P(self.splats.flags), P(self.contributed), lon,
                              ctypes.byref(self.state.planes("m")),
                              ctypes.byref(self.state.planes("v")), ctypes.byref(hp0), d_hp,
                              P(self.status), stream_handle()), "ss_chain_adam")
        self._mark("chain_adam")

    def target_buffer(self, depth: bool = False, slot: int = 0) -> torch.Tensor:
        """The engine's keyframe-target staging buffers ((H, W, 3), or (H, W)
        for the depth target) that the captured graphs read.  step() copies
        its target into slot 0 (stream-ordered, device to device) unless the
        caller passes one of these buffers itself.  There are two RGB slots,
        each with its own graph, so a caller can upload keyframe k + 1 into
        one slot (e.g. from pinned host memory on a copy stream) while step
        k still reads the other: no device-to-device copy per step."""
        if depth:
            if self._tdep_buf is None:
                self._tdep_buf = torch.zeros((self.H, self.W), dtype=torch.float32,
                                             device=self.dev)
            return self._tdep_buf
        if slot not in (0, 1):
            raise ValueError("target slot must be 0 or 1")
        if slot == 1 and self._tgt_buf1 is None:
            self._tgt_buf1 = torch.zeros((self.H, self.W, 3), dtype=torch.float32,
                                         device=self.dev)
        return self._tgt_buf if slot == 0 else self._tgt_buf1

    def upload_target(self, host: torch.Tensor, slot: int, after=None, chunks: int = 4):
        """Upload one keyframe target (H, W, 3) float32 from pinned host
        memory into target slot `slot`, split into row chunks copied
        concurrently on `chunks` copy streams (one pinned host-to-device copy
        of 9.8 MB ran at 22 GB/s on a box where four concurrent chunks ran
        at 34 GB/s; on a fast host both reach ~50).  `after`: an event the
        copies wait for (the slot's previous reader).  Returns the event a
        step reading the slot must wait on (torch.cuda.current_stream()
        .wait_event), or pass the buffer to step() after it."""
        dst = self.target_buffer(slot=slot)
        if tuple(host.shape) != tuple(dst.shape) or host.dtype != torch.float32:
            raise ValueError(f"target must be float32 {tuple(dst.shape)}, got "
                             f"{host.dtype} {tuple(host.shape)}")
        if host.device.type != "cpu" or not host.is_pinned():
            raise ValueError("upload_target needs a pinned host tensor (tensor.pin_memory())")
        k = max(1, min(int(chunks), 8))
        streams = getattr(self, "_copy_streams", None)
        if streams is None or len(streams) < k or streams[0].device != self.dev:
            streams = self._copy_streams = [torch.cuda.Stream(device=self.dev)
                                            for _ in range(k)]
        src, out = host.reshape(self.H, -1), dst.reshape(self.H, -1)
        # events reused per slot (a wait already issued keeps the state it saw)
        evs = getattr(self, "_upload_events", {})
        self._upload_events = evs
        if (slot, k) not in evs:
            evs[(slot, k)] = [torch.cuda.Event() for _ in range(k + 1)]
        done = evs[(slot, k)]
        for i in range(k):
            r0, r1 = i * self.H // k, (i + 1) * self.H // k
            st = streams[i]
            if after is not None:
                st.wait_event(after)
            with torch.cuda.stream(st):
                out[r0:r1].copy_(src[r0:r1], non_blocking=True)
            done[i].record(st)
        for ev in done[1:k]:
            streams[0].wait_event(ev)
        done[k].record(streams[0])
        return done[k]

    def _stage_target(self, rec: StepRecord):
        """(target buffer, depth buffer, slot) the graph of this step reads."""
        slot = 0
        if self._tgt_buf1 is not None and rec.target.data_ptr() == self._tgt_buf1.data_ptr():
            slot = 1
        tgt = self.target_buffer(slot=slot)
        if rec.target.data_ptr() != tgt.data_ptr():
            tgt.copy_(rec.target.reshape(tgt.shape), non_blocking=True)
        tdep = None
        if rec.target_depth is not None:
            tdep = self.target_buffer(depth=True)
            if rec.target_depth.data_ptr() != tdep.data_ptr():
                tdep.copy_(rec.target_depth.reshape(tdep.shape), non_blocking=True)
        return tgt, tdep, slot

    def _run(self, rec: StepRecord):
        self._stage_params(rec)
        if self.use_graph and self.profile is None:
            tgt, tdep, slot = self._stage_target(rec)
            key = (tdep is not None, slot)
            g = self._graphs.get(key)
            if g is None:
                g = self._capture(lambda: self._body(rec.camera, tgt, tdep))
                self._graphs[key] = g
            g.replay()
        else:
            self._body(rec.camera, rec.target, rec.target_depth)
        self.launches += self._launches_per_step()
        self._snapshot(rec)

    def _capture(self, body):
        """Capture body() into a CUDA graph on a side stream.  Not through
        torch.cuda.graph(): its entry empties the device and pinned-host
        allocator caches (and may run gc), so the next allocations go back to
        cudaMalloc / cudaHostAlloc -- tens to hundreds of ms, at every
        re-capture after a densify."""
        torch.cuda.synchronize()
        if getattr(self, "_cap_stream", None) is None or self._cap_stream.device != self.dev:
            self._cap_stream = torch.cuda.Stream(device=self.dev)
        g = torch.cuda.CUDAGraph()
        cs = self._cap_stream
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            g.capture_begin()
            try:
                body()
            finally:
                g.capture_end()
        torch.cuda.current_stream().wait_stream(cs)
        return g

    def _launches_fb(self, depth_loss: bool):
        """Library kernels one _forward_backward enqueues (K1-K7 of a view)."""
        k = KERNELS_PER_CALL["step_fb"] + binning_kernels(self.n_tiles, len(self.gmap))
        if self.n_tiles <= _lib.ORDER_MAX_TILES:
            k += KERNELS_PER_CALL["tile_order"]
        if depth_loss:
            k += 3  # ss_depth_l1
        return k

    def _launches_per_step(self):
        return (self._launches_fb(bool(self.opts.with_depth and self.cfg.depth_weight))
                + KERNELS_PER_CALL["chain_adam"] + KERNELS_PER_CALL["snapshot"])

    def _drain(self, lag: int):
        """Consume status snapshots older than `lag` steps; recover overflow."""
        while len(self._records) > lag:
            rec = self._records[0]
            rec.event.synchronize()
            row = self._host[rec.slot].numpy().copy()
            if int(row[_lib.ST_OVERFLOW]):
                self._recover(int(row[_lib.ST_PAIRS]))
                continue
            self._check_errors(row)
            self._log(rec, row)
            self._records.pop(0)

    def _check_errors(self, row):
        """Raise the reference's error for a status row (api.py:127-129,
        core.py:225-229, optimizer.py:111-113)."""
        if row[_lib.ST_BAD_PARAM] < 2 ** 62:
            raise ValueError(f"non-finite parameter in primitive {int(row[_lib.ST_BAD_PARAM])}")
        if row[_lib.ST_ZERO_QUAT] < 2 ** 62:
            raise ValueError("zero-norm quaternion in map")
        if row[_lib.ST_BAD_GRAD] < 2 ** 62:
            raise FloatingPointError("non-finite gradient (primitive "
                                     f"{int(row[_lib.ST_BAD_GRAD])})")

    def _log(self, rec, row):
        npx = self.H * self.W * 3
        l1 = row[_lib.SN_L1_SUM] / npx
        ssim = row[_lib.SN_SSIM_SUM] / npx
        lam = self.cfg.lambda_ssim
        rendered = (1 - lam) * l1 + lam * (1 - ssim)
        reg = row[_lib.SN_OPACITY_SUM] / max(len(self.gmap), 1)
        self._loss_log.append((rec.index, rendered + self.cfg.lambda_o * reg, rendered))

    def _recover(self, pairs_seen: int):
        """Grow pair buffers and replay every pending (skipped) step in order."""
        torch.cuda.current_stream().synchronize()
        pending = list(self._records)
        self._records.clear()
        newcap = max(int(pairs_seen * self.cfg.pair_margin) + 4096, self._cap * 2)
        self._alloc_pair_buffers(newcap)
        check(lib().ss_status_reset(P(self.status), stream_handle()), "ss_status_reset")
        for rec in pending:
            rec.replayed += 1
            self._run(rec)
        torch.cuda.current_stream().synchronize()
        self._records = pending

    def synchronize(self):
        self._drain(0)
        if self._mv_unchecked:
            # the last keyframe-batch step's Adam may have reported errors
            self._mv_unchecked = False
            self._check_errors(self.status.cpu().numpy())

    def losses(self):
        """(iteration, total loss, rendered loss) of every consumed step."""
        self.synchronize()
        return list(self._loss_log)

    def last_pair_count(self) -> int:
        return int(self.status[_lib.ST_PAIRS].item())

    def fit_capacity(self, cameras, margin: float | None = None):
        """Size the pair buffers for a camera or a list of cameras (one
        binning per camera + one sync, no update).  Only grows the buffers;
        returns the largest pair count seen."""
        cams = cameras if isinstance(cameras, (list, tuple)) else [cameras]
        L = lib()
        s = stream_handle()
        mp, op = self.gmap.ss(), self.opts.to_ss()
        tiny = BinBuffers.alloc(0, self.n_tiles, self.dev)
        ws = bin_workspace(len(self.gmap), 0, self.n_tiles, self.dev)
        sts = torch.empty((len(cams), _lib.STATUS_WORDS), dtype=torch.int64, device=self.dev)
        for k, camera in enumerate(cams):
            cm = Camera.of(camera).to_ss()
            st = sts[k]
            check(L.ss_status_reset(P(st), s), "ss_status_reset")
            check(L.ss_preprocess(ctypes.byref(mp), ctypes.byref(cm), None, ctypes.byref(op),
                                  ctypes.byref(self.splats.ss()), P(st), s), "ss_preprocess")
            check(L.ss_bin_sort(len(self.gmap), ctypes.byref(self.splats.ss()),
                                ctypes.byref(cm), ctypes.byref(tiny.ss()), P(ws), ws.numel(),
                                P(st), s), "ss_bin_sort")
        p = int(sts[:, _lib.ST_PAIRS].max().item()) if cams else 0
        m = self.cfg.pair_margin if margin is None else margin
        want = int(p * m) + 4096
        if want > self._cap:
            self._alloc_pair_buffers(want)
        return p

    # ------------------------------------------------- densify / reset (K10)
    def _maybe_densify(self):
        cfg = self.cfg
        if cfg.densify is not None and self.since_densify >= cfg.densify.interval:
            self.densify()
        if (cfg.opacity_reset_interval and self.iteration > 0
                and self.iteration % cfg.opacity_reset_interval == 0):
            self.synchronize()
            opacity_reset(self.gmap, self.state, cfg.opacity_reset_ceiling)

    @traced("ss.MappingEngine.densify")
    def densify(self, normals=None):
        """densify_and_prune + resize_for_densify as one compaction
        (trainer.py:187-193)."""
        self.synchronize()
        n = len(self.gmap)
        planes = []
        new_m, new_v = {}, {}
        # the engine's moments ride through the compaction as extra planes
        from .densify import densify_count
        _, c, _ = densify_count(self.gmap, self.cfg.densify, self.cfg.scene_extent)
        n_out = int(c[0] + c[4])
        for d, nd in ((self.state.m, new_m), (self.state.v, new_v)):
            for k, t in d.items():
                out = torch.zeros((n_out,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
                planes.append((t.contiguous(), out))
                nd[k] = out
        res = densify_and_prune(self.gmap, self.cfg.densify, self.cfg.scene_extent,
                                normals=normals, rng=None if normals is not None else
                                int(np.random.default_rng(self.iteration).integers(1, 2 ** 62)),
                                extra_planes=planes)
        self.state.m, self.state.v = new_m, new_v
        self.since_densify = 0
        # the map planes and the Adam moments are new tensors whatever the
        # count: captured graphs would replay into freed memory
        self._graphs.clear()
        if len(self.gmap) != n:
            self._alloc_map_buffers()
            # pair buffers only grow: a shrunken map keeps them (no cudaMalloc of
            # hundreds of MB at a prune); the binning workspace is re-sized only
            # if the new map needs more
            need = max(self._cap * len(self.gmap) // max(n, 1), 4096)
            ws = int(lib().ss_bin_workspace_bytes(len(self.gmap), self._cap, self.n_tiles))
            if need > self._cap:
                self._alloc_pair_buffers(need)
            elif ws > self.bin_ws.numel():
                self.bin_ws = None
                self.bin_ws = bin_workspace(len(self.gmap), self._cap, self.n_tiles, self.dev)
        return res

    def add_points(self, points, colors):
        """A keyframe's point cloud enters the map (trainer.py:160-174):
        seed_from_points on the GPU, insert, Adam moments grown with zeros
        (resize_for_densify with every old primitive surviving)."""
        from .densify import seed_from_points
        self.synchronize()
        pos, rot, ls, opl, sh = seed_from_points(points, colors, self.cfg.scene_extent,
                                                 self.dev)
        n_new = int(pos.shape[0])
        if n_new == 0:
            return 0
        n = len(self.gmap)
        self.gmap.insert_device(pos, rot, ls, opl, sh[:, 0, :])
        for d in (self.state.m, self.state.v):
            for k, t in list(d.items()):
                z = torch.zeros((n_new,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
                d[k] = torch.cat([t, z]).contiguous()
        self._alloc_map_buffers()
        self._alloc_pair_buffers(max(self._cap * len(self.gmap) // max(n, 1), 4096))
        return n_new

    # ------------------------------------------------------- multi-view
    def _flat_grads(self):
        """The flat per-Gaussian buffer of a keyframe-batch step (layout:
        distributed.flat_layout) and its ss_param_grads view."""
        from .distributed import flat_layout
        n = len(self.gmap)
        if self._flat is None or self._flat_n != n:
            layout, total = flat_layout(max(n, 1), self.opts.sh_degree)
            self._flat = torch.zeros(total, dtype=torch.float32, device=self.dev)
            self._flat_n = n
            views = {name: self._flat[off:off + k * max(n, 1)] for name, k, off in layout}
            self._fv = views
            self._flat_tail = self._flat[total - 2:]
            g = _lib.SSParamGrads()
            g.d_position, g.d_rotation = P(views["position"]), P(views["rotation"])
            g.d_log_scale, g.d_opacity = P(views["log_scale"]), P(views["opacity"])
            g.d_sh_dc, g.d_sh_rest = P(views["sh_dc"]), P(views["sh_rest"])
            g.d_pos2d_norm = P(views["pos2d"])
            g.d_stat_g2d, g.d_stat_g3d, g.d_stat_cnt = (P(views["stat_g2d"]),
                                                        P(views["stat_g3d"]),
                                                        P(views["stat_cnt"]))
            self._fss = g
            self._mv_host = torch.zeros(_lib.STATUS_WORDS + 1, dtype=torch.int64,
                                        pin_memory=True)
        return self._flat, self._fss

    @traced("ss.MappingEngine.multiview_step")
    def multiview_step(self, cameras, targets, target_depths=None, allreduce=None,
                       add_reg: bool = True):
        """Keyframe batch: the sum of per-view gradients
        (+ the opacity-reg gradient once, add_reg on one rank), an optional
        all-reduce of the flat buffer, then Adam and the statistics update.

        Every view is enqueued without a host sync.  ss_status_flags writes
        this rank's overflow / error flags into the buffer's tail, so after
        the (optional) all-reduce ONE host read tells every rank whether any
        rank overflowed its pair buffers -- then all ranks redo the step
        together with grown buffers (nothing was applied yet) -- or hit an
        error -- then every rank raises before Adam touches the map."""
        self._maybe_densify()
        # pending single-view steps apply first, in order (errors of the last
        # batch step's Adam are sticky: this step's status read raises them)
        self._drain(0)
        L = lib()
        s = stream_handle()
        n = len(self.gmap)
        flat, fss = self._flat_grads()
        lon = float(self.cfg.lambda_o / n) if (n and add_reg) else 0.0
        views = [(Camera.of(c), t, target_depths[v] if target_depths is not None else None)
                 for v, (c, t) in enumerate(zip(cameras, targets))]

        def run_views(sync_each: bool):
            flat.zero_()
            losses = []
            for v, (cam, tgt, td) in enumerate(views):
                depth_loss = bool(self.opts.with_depth and td is not None
                                  and self.cfg.depth_weight != 0.0)
                while True:
                    mp, cm, op = self._forward_backward(cam, tgt, td, v)
                    self.launches += self._launches_fb(depth_loss)
                    if not sync_each:
                        break
                    row = self.status.cpu().numpy()
                    if not int(row[_lib.ST_OVERFLOW]):
                        break
                    # redo path: grow to this view's pair count, run it again
                    self._alloc_pair_buffers(max(
                        self._cap, int(int(row[_lib.ST_PAIRS]) * self.cfg.pair_margin) + 4096))
                    check(L.ss_status_reset(P(self.status), s), "ss_status_reset")
                    self.launches += 1
                check(L.ss_chain_backward(ctypes.byref(mp), ctypes.byref(cm), ctypes.byref(op),
                                          P(self.g2d), P(self.splats.flags),
                                          P(self.contributed), lon if v == 0 else 0.0,
                                          _lib.SS_CHAIN_ACCUMULATE | _lib.SS_CHAIN_STAT_PLANES,
                                          ctypes.byref(fss), P(self.status), s),
                      "ss_chain_backward")
                self.launches += 1
                losses.append(self.sums[:2].clone())
            check(L.ss_status_flags(P(self.status), P(self._flat_tail), s), "ss_status_flags")
            self.launches += 1
            if allreduce is not None:
                allreduce(flat)
            # one host read: this rank's status row + the (reduced) flags
            h = self._mv_host
            h[:_lib.STATUS_WORDS].copy_(self.status, non_blocking=True)
            h[_lib.STATUS_WORDS:].view(torch.float32).copy_(self._flat_tail, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            row = h[:_lib.STATUS_WORDS].numpy().copy()
            flags = h[_lib.STATUS_WORDS:].view(torch.float32).numpy().copy()
            return losses, row, flags

        losses, row, flags = run_views(sync_each=False)
        if flags[0] > 0:
            # some rank overflowed: every rank redoes the step, view by view
            # with a read per view (the rare path), so the collectives match
            check(L.ss_status_reset(P(self.status), s), "ss_status_reset")
            self.launches += 1
            losses, row, flags = run_views(sync_each=True)
        if flags[1] > 0:
            self._check_errors(row)
            raise FloatingPointError("non-finite value reported by another rank of the "
                                     "keyframe-sharded step")
        self.state.step_count += 1
        hp = self.state.hparams(self.opts.sh_degree > 0)
        mp = self.gmap.ss()
        check(L.ss_adam_step(ctypes.byref(mp), ctypes.byref(fss),
                             ctypes.byref(self.state.planes("m")),
                             ctypes.byref(self.state.planes("v")), ctypes.byref(hp),
                             P(self.status), s), "ss_adam_step")
        check(L.ss_apply_stat_planes(ctypes.byref(mp), ctypes.byref(fss), s),
              "ss_apply_stat_planes")
        self.launches += 2  # Adam + statistics planes
        self._mv_unchecked = True
        self.iteration += 1
        self.since_densify += 1
        return losses
