"""Work statistics of the splat-wise backward (diagnostics): after PROF_ITERS
training iterations on the bench workload (S(300k), 1200x680; 250 = the
bench's `converged` block), per (tile, 64-position unit) of the forward's
list: the active pixels (a blend bit set in either bucket: the unit's
wavefront length), the wavefront steps (pairs + 15 ramp), the executed
(pixel, splat) term slots (steps x 32 lanes x 2 splats x 2 pixels) and the
useful ones (blend bits set, popcount of the checkpoint masks).

    PROF_ITERS=250 python tools/bwd_stats.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

n = int(os.environ.get("PROF_N", 300000))
W = int(os.environ.get("PROF_W", 1200))
H = int(os.environ.get("PROF_H", 680))
iters = int(os.environ.get("PROF_ITERS", 250))
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=0)
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam, opts).image
eng = ss.MappingEngine(ss.GaussianMap.from_scene(survey_scene(n, 0)), W, H, opts)
eng.fit_capacity(cam)
eng.enable_graph()
for _ in range(iters):
    eng.step(cam, tgt)
eng.synchronize()
out = ss.rasterize_forward(eng.gmap, cam, opts)
torch.cuda.synchronize()
nc = out.n_contrib.cpu().numpy().astype(np.int64)
ke = out.k_eff_tiles.cpu().numpy().astype(np.int64)
base = out.bins.ckpt_base.cpu().numpy().astype(np.int64)
mask = out.ckpt_mask.cpu().numpy().view(np.uint32)
pc = np.unpackbits(mask.view(np.uint8)).reshape(-1, 32).sum(1).astype(np.int64)
tx, ty = (W + 15) // 16, (H + 15) // 16
pad = np.zeros((ty * 16, tx * 16), np.int64)
pad[:H, :W] = nc
tiles_nc = pad.reshape(ty, 16, tx, 16).transpose(0, 2, 1, 3).reshape(tx * ty, 256)


units = []
useful = executed = steps_total = ramp_total = 0
pairs_hist = []
band_pos, band_pairs = [], []
for t in range(tx * ty):
    nu = (ke[t] + 63) // 64
    for u in range(nu):
        s0 = (base[t] + 2 * u) * 256
        live0 = tiles_nc[t] > 64 * u
        live1 = tiles_nc[t] > 64 * u + 32
        has1 = 2 * u + 1 < (ke[t] + 31) // 32
        m0 = np.where(live0, mask[s0:s0 + 256], 0)
        m1 = np.where(live1, mask[s0 + 256:s0 + 512], 0) if has1 else 0 * m0
        p0 = np.where(live0, pc[s0:s0 + 256], 0)
        p1 = np.where(live1, pc[s0 + 256:s0 + 512], 0) if has1 else 0 * p0
        act = (m0 | m1) != 0
        npair = (int(act.sum()) + 1) // 2
        # per 4-row band: positions blended by any of its pixels (both buckets)
        for b in range(4):
            o0 = np.bitwise_or.reduce(m0[64 * b:64 * (b + 1)].astype(np.uint64))
            o1 = np.bitwise_or.reduce(m1[64 * b:64 * (b + 1)].astype(np.uint64))
            npos = bin(int(o0)).count("1") + bin(int(o1)).count("1")
            band_pos.append(npos)
            band_pairs.append((int(act[64 * b:64 * (b + 1)].sum()) + 1) // 2)
        st = npair + 15
        useful += int(p0.sum() + p1.sum())
        executed += st * 32 * 2 * 2
        steps_total += st
        ramp_total += 15
        pairs_hist.append(npair)
ph = np.array(pairs_hist)
print(json.dumps({
    "iterations": iters, "units": len(ph), "pairs": int(out.pair_count),
    "mean_active_pairs_per_unit": float(ph.mean()), "p50_pairs": float(np.median(ph)),
    "p10_pairs": float(np.percentile(ph, 10)), "p90_pairs": float(np.percentile(ph, 90)),
    "wavefront_steps": steps_total, "ramp_share_of_steps": ramp_total / steps_total,
    "term_slots_executed": executed, "term_slots_useful": useful,
    "useful_fraction": useful / executed,
    "mean_sigma": float(torch.sigmoid(eng.gmap.opacity_logits).mean()),
    "band_positions_mean": float(np.mean(band_pos)),
    "band_positions_hist_le16_le32_le48_le64": [float(np.mean(np.array(band_pos) <= v))
                                                for v in (16, 32, 48, 64)],
    "band_pairs_mean": float(np.mean(band_pairs)),
}))
