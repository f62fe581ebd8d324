"""Per-CTA timeline of the forward blend at the bench workload (diagnostics).

Needs the library built with -DSS_FWD_TRACE, e.g. on the GPU box:
    make -C paper_2410_00486_b200/csrc clean
    make -C paper_2410_00486_b200/csrc FLAGS+=-DSS_FWD_TRACE
    python tools/trace_forward.py
Prints the SM-busy fraction of the forward (sum of CTA durations / (148 x
elapsed x resident CTAs)), when the last CTAs start and end, and how the
CTA duration relates to the tile's list length and k_eff."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200 import _lib  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

n = int(os.environ.get("PROF_N", 300000))
W = int(os.environ.get("PROF_W", 1200))
H = int(os.environ.get("PROF_H", 680))
steps = int(os.environ.get("PROF_STEPS", 10))
g = ss.GaussianMap.from_scene(survey_scene(n, 0))
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=0)
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam, opts).image
eng = ss.MappingEngine(g, W, H, opts)
eng.fit_capacity(cam)
for _ in range(steps):
    eng.step(cam, tgt)
eng.synchronize()
L = _lib.lib()
fn = L.ss_debug_fwd_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
tx, ty = (W + 15) // 16, (H + 15) // 16
T = tx * ty
buf = np.zeros(4 * T, np.uint64)
assert fn(buf.ctypes.data, buf.nbytes) == 0
tr = buf.reshape(T, 4).astype(np.int64)
sm, t0, t1 = tr[:, 1], tr[:, 2], tr[:, 3]
base = t0.min()
t0, t1 = t0 - base, t1 - base
dur = t1 - t0
el = t1.max()
k_eff = eng.k_eff.cpu().numpy().astype(np.int64)
lens = (eng.bins.tile_end.cpu().numpy().astype(np.int64)
        - eng.bins.tile_start.cpu().numpy().astype(np.int64))
ft = eng.final_t.cpu().numpy() if hasattr(eng, "final_t") else None
iters = tr[:, 0]
c = np.corrcoef(np.stack([dur, lens, k_eff, iters]).astype(np.float64))
print(f"corr(dur, len) {c[0, 1]:.3f}  corr(dur, k_eff) {c[0, 2]:.3f}  "
      f"corr(dur, warp iterations) {c[0, 3]:.3f}")
np.savez("gpurun_out/fwd_trace_meta.npz", lens=lens, k_eff=k_eff, iters=iters)
print(f"tiles {T}  elapsed {el / 1e3:.1f} us  mean CTA {dur.mean() / 1e3:.2f} us  "
      f"max CTA {dur.max() / 1e3:.2f} us  sum {dur.sum() / 1e3:.0f} us")
nsm = int(sm.max()) + 1
busy = np.zeros(nsm)
last = np.zeros(nsm)
for s_ in range(nsm):
    m = sm == s_
    if m.any():
        last[s_] = t1[m].max()
        busy[s_] = dur[m].sum()
print(f"SM last-end: min {last.min() / 1e3:.1f} median {np.median(last) / 1e3:.1f} "
      f"max {last.max() / 1e3:.1f} us")
order = np.argsort(t0)
print("last 10 CTAs to start (tile, start us, dur us):")
for i in order[-10:]:
    print(f"  {i:5d} {t0[i] / 1e3:7.1f} {dur[i] / 1e3:7.1f}")
print("longest 10 CTAs (tile, start us, dur us):")
for i in np.argsort(dur)[-10:]:
    print(f"  {i:5d} {t0[i] / 1e3:7.1f} {dur[i] / 1e3:7.1f}")
# ideal: LPT list scheduling of the measured durations on nsm x 9 slots
import heapq  # noqa: E402
for name, seq in (("raster", np.arange(T)), ("len desc", None), ("k_eff desc", np.argsort(-k_eff)),
                  ("iters desc", np.argsort(-iters)), ("dur desc", np.argsort(-dur))):
    if seq is None:
        seq = np.argsort(-lens, kind="stable")
    h = [0.0] * (nsm * 9)
    for i in seq:
        v = heapq.heappop(h)
        heapq.heappush(h, v + dur[i] * 1.0)
    print(f"greedy {name:10s}: makespan {max(h) / 1e3:.1f} us (slot model, 9 CTAs/SM)")
np.save("gpurun_out/fwd_trace.npy", tr)
# predictor stability: the next iteration's CTA durations ordered by this one's
eng.step(cam, tgt)
eng.synchronize()
buf2 = np.zeros(4 * T, np.uint64)
assert fn(buf2.ctypes.data, buf2.nbytes) == 0
tr2 = buf2.reshape(T, 4).astype(np.int64)
dur2 = tr2[:, 3] - tr2[:, 2]
print(f"next iteration: corr(dur, dur_prev) {np.corrcoef(dur, dur2)[0, 1]:.3f}")
for name, seq in (("raster", np.arange(T)), ("prev dur", np.argsort(-dur)),
                  ("prev iters", np.argsort(-iters)), ("own dur", np.argsort(-dur2))):
    h = [0.0] * (nsm * 9)
    for i in seq:
        v = heapq.heappop(h)
        heapq.heappush(h, v + dur2[i] * 1.0)
    print(f"next iteration, order {name:10s}: makespan {max(h) / 1e3:.1f} us")
# SSIM kernels (same diagnostics build)
if hasattr(L, "ss_debug_ssim_trace"):
    f2 = L.ss_debug_ssim_trace
    f2.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    nb = ((W + 31) // 32) * ((H + 31) // 32)
    for kind, name in ((0, "ssim_fwd"), (1, "ssim_bwd")):
        b3 = np.zeros(4 * nb, np.uint64)
        assert f2(kind, b3.ctypes.data, b3.nbytes) == 0
        t3 = b3.reshape(nb, 4).astype(np.int64)
        s3, a3, e3 = t3[:, 1], t3[:, 2] - t3[:, 2].min(), t3[:, 3] - t3[:, 2].min()
        d3 = e3 - a3
        lastend = np.array([e3[s3 == k].max() for k in np.unique(s3)])
        nper = np.bincount(s3)
        print(f"{name}: CTAs {nb} elapsed {e3.max() / 1e3:.1f} us, CTA dur mean "
              f"{d3.mean() / 1e3:.2f} min {d3.min() / 1e3:.2f} max {d3.max() / 1e3:.2f} us, "
              f"SM last-end min {lastend.min() / 1e3:.1f} median {np.median(lastend) / 1e3:.1f}, "
              f"CTAs/SM {nper[nper > 0].min()}..{nper.max()}, start of last CTA "
              f"{a3.max() / 1e3:.1f} us")
        np.save(f"gpurun_out/{name}_trace.npy", t3)
