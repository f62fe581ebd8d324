"""Warm per-kernel device times of the fused mapping iteration (CUPTI via
torch.profiler: no cache flush, no serialisation -- unlike an ncu launch
list).  Prints one row per kernel name: mean us per step, launches per step."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

n = int(os.environ.get("PROF_N", 300000))
W = int(os.environ.get("PROF_W", 1200))
H = int(os.environ.get("PROF_H", 680))
steps = int(os.environ.get("PROF_STEPS", 10))
g = ss.GaussianMap.from_scene(survey_scene(n, 0))
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=int(os.environ.get("PROF_DEG", 0)))
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam, opts).image
eng = ss.MappingEngine(g, W, H, opts)
eng.fit_capacity(cam)
for _ in range(int(os.environ.get("PROF_WARM", 5))):
    eng.step(cam, tgt)
eng.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        eng.step(cam, tgt)
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.split("(")[0].replace("void ", "")
        tot[name] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        cnt[name] += 1
allsum = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / steps:9.1f} us/step  x{cnt[k] / steps:4.1f}  {100 * v / allsum:5.1f}%  {k[:90]}")
print(f"kernel time per step {allsum / steps:.1f} us")
