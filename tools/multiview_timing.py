"""Throughput of MappingEngine.multiview_step (keyframe batch of 8 views, 1M Gaussians)
on one GPU -- the single-GPU case of BASELINE configs[3] (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2410_00486_b200 as ss
from paper_2410_00486_b200.scene import survey_camera, survey_scene
n, W, H, V = 1000000, 1200, 680, 8
g = ss.GaussianMap.from_scene(survey_scene(n, 0))
opts = ss.RasterOpts(sh_degree=0)
cams = [survey_camera(W, H, v, V) for v in range(V)]
tm = ss.GaussianMap.from_scene(survey_scene(n, 100))
tg = [ss.rasterize_forward(tm, c, opts).image.clone() for c in cams]
del tm
eng = ss.MappingEngine(g, W, H, opts)
for c in cams:
    eng.fit_capacity(c)
for _ in range(2):
    eng.multiview_step(cams, tg)
torch.cuda.synchronize()
t = time.perf_counter()
K = 5
for _ in range(K):
    eng.multiview_step(cams, tg)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / K
print(f"multiview_step 1M x {V} views on 1 GPU: {dt*1e3:.2f} ms/step, {V/dt:.0f} views/s")
