"""Distribution of the splat-wise backward's work units at the bench
workload: per (tile, 64-position unit), the pixels still blending at the
unit start (n_contrib > 64 u) -- the length of the unit's wavefront, whose
ramp costs 31 steps regardless of it (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

n = int(os.environ.get("PROF_N", 300000))
W = int(os.environ.get("PROF_W", 1200))
H = int(os.environ.get("PROF_H", 680))
steps = int(os.environ.get("PROF_STEPS", 6))
g = ss.GaussianMap.from_scene(survey_scene(n, 0))
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=0)
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam, opts).image
eng = ss.MappingEngine(g, W, H, opts)
eng.fit_capacity(cam)
for _ in range(steps):
    eng.step(cam, tgt)
eng.synchronize()
out = ss.rasterize_forward(eng.gmap, cam, opts)
nc = out.n_contrib.cpu().numpy().astype(np.int64)
tx, ty = (W + 15) // 16, (H + 15) // 16
pad = np.zeros((ty * 16, tx * 16), np.int64)
pad[:H, :W] = nc
tiles = pad.reshape(ty, 16, tx, 16).transpose(0, 2, 1, 3).reshape(ty * tx, 256)
kmax = tiles.max(1)
units = []
for t in range(tiles.shape[0]):
    for u in range((kmax[t] + 63) // 64):
        units.append(int((tiles[t] > 64 * u).sum()))
units = np.array(units)
pairs = (units + 1) // 2
print(f"units {len(units)}  mean active px {units.mean():.1f}  median {np.median(units):.0f}")
for lo, hi in [(0, 16), (16, 32), (32, 64), (64, 128), (128, 192), (192, 257)]:
    m = (units >= lo) & (units < hi)
    print(f"  active px [{lo:3d},{hi:3d}): {m.sum():6d} units, steps {(pairs[m] + 31).sum():8d} "
          f"(ramp share {31 * m.sum() / max((pairs[m] + 31).sum(), 1):.2f})")
print(f"total steps {(pairs + 31).sum()}  ramp steps {31 * len(units)}")
