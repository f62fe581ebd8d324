"""Stage-by-stage timing/debug run at increasing map sizes (GPU)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_00486_b200 as ss
from paper_2410_00486_b200 import _lib
from paper_2410_00486_b200.scene import survey_scene, survey_camera

def log(*a):
    print(*a, flush=True)

for n, W, H in [(10000, 128, 96), (50000, 640, 480), (150000, 640, 480), (300000, 1200, 680)]:
    t0 = time.time()
    g = ss.GaussianMap.from_scene(survey_scene(n, 0))
    cam = survey_camera(W, H)
    opts = ss.RasterOpts(sh_degree=0)
    torch.cuda.synchronize(); log(n, "map", time.time() - t0)
    out = ss.rasterize_forward(g, cam, opts)
    torch.cuda.synchronize(); log(n, "fwd", time.time() - t0, "P", out.pair_count,
                                  "status", out.status.cpu().tolist())
    tgt = out.image.clone() * 0.9
    lb = ss.compute_losses(out.image, tgt, g.opacity_logits)
    torch.cuda.synchronize(); log(n, "loss", time.time() - t0, lb.total)
    gr = ss.backward_splatwise(out, lb.grad_image)
    torch.cuda.synchronize(); log(n, "bwd", time.time() - t0, float(gr.position.abs().max()))
    eng = ss.MappingEngine(g, W, H, opts)
    p = eng.fit_capacity(cam)
    torch.cuda.synchronize(); log(n, "fit", time.time() - t0, p, eng.pair_capacity)
    for k in range(3):
        eng.step(cam, tgt)
        torch.cuda.synchronize(); log(n, "step", k, time.time() - t0)
    eng.synchronize()
    t1 = time.time()
    for k in range(10):
        eng.step(cam, tgt)
    eng.synchronize()
    log(n, "10 steps", (time.time() - t1) / 10 * 1000, "ms/step", eng.losses()[-1])
