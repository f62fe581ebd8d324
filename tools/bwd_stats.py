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
quad_steps = 0  # per-quadrant chains (see below)
seg_steps = 0
seg_need = seg_have = 0
GROUPS = [(8, 8), (16, 4), (8, 4), (4, 8), (4, 4), (16, 2), (8, 2)]
grp_stats = {}
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
        # quadrant chains: per 8x8 quadrant the positions blended by any of its
        # pixels (both buckets) and its active column pairs; a chain of n <= 32
        # positions runs np + ceil(n/2) - 1 steps in a half-warp, n > 32 splits
        # at the bucket boundary; jobs sorted by length, paired per round
        jobs = []  # (active pairs, positions) per chain
        a2 = act.reshape(8, 2, 16)  # (c, row parity, col)
        for q in range(4):
            rows = slice(0, 8) if q < 2 else slice(8, 16)
            cols = slice(0, 8) if q % 2 == 0 else slice(8, 16)
            mq0 = m0.reshape(16, 16)[rows, cols].astype(np.uint64)
            mq1 = m1.reshape(16, 16)[rows, cols].astype(np.uint64)
            o0 = int(np.bitwise_or.reduce(mq0.ravel()))
            o1 = int(np.bitwise_or.reduce(mq1.ravel()))
            n0, n1 = bin(o0).count("1"), bin(o1).count("1")
            cq = slice(0, 4) if q < 2 else slice(4, 8)
            npq = int((a2[cq, 0, cols] | a2[cq, 1, cols]).sum())
            if n0 + n1 == 0:
                continue
            if n0 + n1 <= 32:
                jobs.append((npq, n0 + n1))
            else:
                jobs.append((npq, n0))
                if n1:
                    jobs.append((npq, n1))
        stp = sorted((p + (n + 1) // 2 - 1 for p, n in jobs), reverse=True)
        quad_steps += sum(stp[0::2])
        # segments: chains (2 positions per lane) packed first-fit-decreasing
        # into rounds of 32 lanes; a round runs max(np + L - 1) steps
        rounds = []
        for p, n in sorted(jobs, key=lambda j: -(j[0] + (j[1] + 1) // 2)):
            L = (n + 1) // 2
            for r in rounds:
                if r[0] + L <= 32:
                    r[0] += L
                    r[1] = max(r[1], p + L - 1)
                    break
            else:
                rounds.append([L, p + L - 1])
        seg_steps += sum(r[1] for r in rounds)
        # lane-steps the chains need vs the rounds' 32 lanes x longest chain
        seg_need += sum((p + (n + 1) // 2 - 1) * ((n + 1) // 2) for p, n in jobs)
        seg_have += 32 * sum(r[1] for r in rounds)
        # the same packing for other pixel-group shapes (gw columns x gh rows)
        M0 = m0.reshape(16, 16).astype(np.uint64)
        M1 = m1.reshape(16, 16).astype(np.uint64)
        A = act.reshape(16, 16)
        for (gw, gh) in GROUPS:
            chains = []
            for gy in range(0, 16, gh):
                for gx in range(0, 16, gw):
                    o0 = int(np.bitwise_or.reduce(M0[gy:gy + gh, gx:gx + gw].ravel()))
                    o1 = int(np.bitwise_or.reduce(M1[gy:gy + gh, gx:gx + gw].ravel()))
                    n0, n1 = bin(o0).count("1"), bin(o1).count("1")
                    if n0 + n1 == 0:
                        continue
                    aa = A[gy:gy + gh, gx:gx + gw].reshape(gh // 2, 2, gw)
                    npg = int((aa[:, 0] | aa[:, 1]).sum())
                    if n0 + n1 <= 32:
                        chains.append((npg, n0 + n1))
                    else:
                        chains.append((npg, n0))
                        if n1:
                            chains.append((npg, n1))
            rr = []
            for pp, nn in sorted(chains, key=lambda j: -(j[0] + (j[1] + 1) // 2)):
                L = (nn + 1) // 2
                for r in rr:
                    if r[0] + L <= 32:
                        r[0] += L
                        r[1] = max(r[1], pp + L - 1)
                        break
                else:
                    rr.append([L, pp + L - 1])
            g = grp_stats.setdefault((gw, gh), [0, 0, 0, 0])
            g[0] += sum(r[1] for r in rr)
            g[1] += len(rr)
            g[2] += len(chains)
            g[3] += sum(nn for _, nn in chains)
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
    "quadrant_chain_steps": quad_steps, "quadrant_vs_wavefront": quad_steps / steps_total,
    "segment_rounds_steps": seg_steps, "segments_vs_wavefront": seg_steps / steps_total,
    "segment_lane_utilisation": seg_need / max(seg_have, 1),
    "groups": {"%dx%d" % k: {"vs_wavefront": round(v[0] / steps_total, 4),
                             "rounds_per_unit": round(v[1] / len(ph), 2),
                             "chains_per_unit": round(v[2] / len(ph), 2),
                             "positions_per_chain": round(v[3] / max(v[2], 1), 1)}
               for k, v in grp_stats.items()},
}))
