"""Two fused mapping iterations at the bench workload inside a
cudaProfilerStart/Stop window (for `ncu --profile-from-start off`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

n = int(os.environ.get("PROF_N", 300000))
W = int(os.environ.get("PROF_W", 1200))
H = int(os.environ.get("PROF_H", 680))
steps = int(os.environ.get("PROF_STEPS", 2))
g = ss.GaussianMap.from_scene(survey_scene(n, 0))
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=int(os.environ.get("PROF_DEG", 0)))
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam, opts).image
eng = ss.MappingEngine(g, W, H, opts)
eng.fit_capacity(cam)
eng.enable_graph()
for _ in range(int(os.environ.get("PROF_WARM", 3))):  # 250: the bench's converged regime
    eng.step(cam, tgt)
eng.enable_graph(False)
eng.synchronize()
torch.cuda.profiler.start()
for _ in range(steps):
    eng.step(cam, tgt)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
eng.synchronize()
print("ok", eng.losses()[-1])
