"""Host time of one MappingEngine.step() call (Python + launch, the GPU
idle before the call) and of the bench's e2e loop body, at the bench
workload -- the e2e loop is host-bound when this exceeds the device step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

W, H, n = 1200, 680, 300000
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=0)
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam, opts).image
eng = ss.MappingEngine(ss.GaussianMap.from_scene(survey_scene(n, 0)), W, H, opts)
eng.fit_capacity(cam)
eng.enable_graph()
for _ in range(5):
    eng.step(cam, tgt)
eng.synchronize()
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.step(cam, tgt)
    ts.append(time.perf_counter() - t0)
ts.sort()
print(f"host time per step() call: median {ts[10]*1e6:.1f} us, min {ts[0]*1e6:.1f} us")
if os.environ.get("PROFILE"):
    import cProfile
    import pstats
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        eng.step(cam, tgt)
    pr.disable()
    eng.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)

if os.environ.get("TIMELINE"):
    # device timeline of pipelined steps: gaps between consecutive GPU ops
    from torch.profiler import ProfilerActivity, profile
    eng.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(20):
            eng.step(cam, tgt)
        eng.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    gaps = {}
    prev = None
    for e in evs:
        if prev is not None:
            g = e.time_range.start - prev.time_range.end
            if g > 1.0:
                key = (prev.name[:40], e.name[:40])
                gaps.setdefault(key, []).append(g)
        prev = e
    span = (evs[-1].time_range.end - t0) / 20
    busy = sum(e.time_range.end - e.time_range.start for e in evs) / 20
    print(f"per step: span {span:.1f} us, summed op time {busy:.1f} us")
    for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1]))[:12]:
        print(f"  gap {sum(v)/20:7.2f} us/step  x{len(v):3d}  {k[0]} -> {k[1]}")

if os.environ.get("E2E"):
    # the bench's e2e loop (pinned host upload on a copy stream, double
    # buffered) under the profiler: per-step span and the largest gaps
    from torch.profiler import ProfilerActivity, profile
    sys.argv = [sys.argv[0]]
    import bench  # noqa: E402
    eng.synchronize()
    r = bench.e2e_single(torch, eng, cam, tgt, 20)
    print("e2e (no profiler)", round(r["value"], 1), "it/s")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        bench.e2e_single(torch, eng, cam, tgt, 20)
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    main = [e for e in evs if "HtoD (Pinned" not in e.name or e.time_range.end - e.time_range.start < 50]
    t0 = evs[0].time_range.start
    print(f"per step span {(evs[-1].time_range.end - t0) / 20:.1f} us")
    for e in evs[:0]:
        pass
    big = [e for e in evs if "Memcpy" in e.name]
    for e in big[:12]:
        print(f"  {e.name[:40]:40s} start {e.time_range.start - t0:9.1f} dur {e.time_range.end - e.time_range.start:7.1f}")
    gaps = {}
    prev = None
    for e in evs:
        if prev is not None and "HtoD (Pinned" not in e.name and "HtoD (Pinned" not in prev.name:
            g = e.time_range.start - prev.time_range.end
            if g > 1.0:
                gaps.setdefault((prev.name[:40], e.name[:40]), []).append(g)
        prev = e
    for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1]))[:10]:
        print(f"  gap {sum(v)/20:7.2f} us/step  x{len(v):3d}  {k[0]} -> {k[1]}")
