"""Per-iteration time of the reference-shaped Python API path (rasterize_forward +
compute_losses + backward_splatwise + adam_step + accumulate_grad_stats) at the bench
workload, and a torch.profiler table of one iteration (host syncs, launches)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2410_00486_b200 as ss
from paper_2410_00486_b200.scene import survey_camera, survey_scene
n, W, H = 300000, 1200, 680
g = ss.GaussianMap.from_scene(survey_scene(n, 0))
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=0)
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam, opts).image
st = ss.AdamState.for_map(g)
def it():
    out = ss.rasterize_forward(g, cam, opts)
    lb = ss.compute_losses(out.image, tgt, g.opacity_logits)
    gr = ss.backward_splatwise(out, lb.grad_image)
    gr.opacity_logit += lb.grad_opacity_logit
    ss.adam_step(g, gr, st)
    ss.accumulate_grad_stats(g, gr)
    return lb.total  # the scheduler's loss feed (trainer.py:209)
def timed(mode):
    ss.set_error_mode(mode)
    for _ in range(3): it()
    torch.cuda.synchronize()
    t = time.perf_counter()
    K = 20
    for _ in range(K): it()
    torch.cuda.synchronize()
    ss.check_errors()
    dt = (time.perf_counter() - t) / K
    print(f"API path, {mode} errors (rasterize_forward + compute_losses + backward_splatwise + "
          f"adam_step + stats, loss read each iteration): {dt*1e3:.3f} ms/it, {1/dt:.0f} it/s")
    ss.set_error_mode("eager")
timed("eager")
timed("deferred")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as p:
    it(); torch.cuda.synchronize()
print(p.key_averages().table(sort_by="self_cpu_time_total", row_limit=12))
# device kernels of one iteration, by time
evs = [e for e in p.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
span = evs[-1].time_range.end - evs[0].time_range.start
busy = {}
for e in evs:
    busy.setdefault(e.name[:70], []).append(e.time_range.end - e.time_range.start)
print(f"one iteration: device span {span:.1f} us, {len(evs)} device ops")
for k, v in sorted(busy.items(), key=lambda kv: -sum(kv[1]))[:30]:
    print(f"  {sum(v):8.1f} us  x{len(v):2d}  {k}")
gaps = []
for a, b in zip(evs[:-1], evs[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 5:
        gaps.append((g, a.name[:40], b.name[:40]))
gaps.sort(reverse=True)
print("largest gaps:")
for g in gaps[:10]:
    print(f"  {g[0]:8.1f} us  {g[1]} -> {g[2]}")
