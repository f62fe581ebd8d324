"""Where the e2e step time goes on this box: the keyframe upload alone, the
device step alone, and the upload's duration while steps run (events on the
copy streams), for the bench workload.  python tools/e2e_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

W, H, N = 1200, 680, 300000
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=0)
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(N, 100)), cam, opts).image
eng = ss.MappingEngine(ss.GaussianMap.from_scene(survey_scene(N, 0)), W, H, opts)
eng.fit_capacity(cam)
eng.enable_graph()
host = tgt.cpu().pin_memory()
for k in range(6):
    eng.step(cam, eng.target_buffer(slot=k % 2))
eng.synchronize()
for chunks in (1, 4):
    # upload alone
    t0 = time.perf_counter()
    for k in range(20):
        ev = eng.upload_target(host, k % 2, chunks=chunks)
        ev.synchronize()
    up = (time.perf_counter() - t0) / 20
    print(f"chunks {chunks}: upload alone {up * 1e6:.0f} us ({host.numel() * 4 / up / 1e9:.1f} GB/s)")
# step alone
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(20):
    eng.step(cam, eng.target_buffer(slot=k % 2))
eng.synchronize()
st = (time.perf_counter() - t0) / 20
print(f"step alone (wall) {st * 1e6:.0f} us")
# upload while steps run: time each upload with events on stream 0 of the copy set
main = torch.cuda.current_stream()
cons = [torch.cuda.Event(), torch.cuda.Event()]
for e in cons:
    e.record(main)
ups = [eng.upload_target(host, b, after=cons[b]) for b in range(2)]
durs = []
t0 = time.perf_counter()
for k in range(2, 42):
    b = k % 2
    main.wait_event(ups[b])
    eng.step(cam, eng.target_buffer(slot=b))
    cons[b].record(main)
    s_ev = torch.cuda.Event(enable_timing=True)
    e_ev = torch.cuda.Event(enable_timing=True)
    cs = eng._copy_streams[0]
    cs.wait_event(cons[b])
    s_ev.record(cs)
    ups[b] = eng.upload_target(host, b, after=cons[b])
    e_ev.record(cs)
    durs.append((s_ev, e_ev))
eng.synchronize()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 40
d = sorted(s.elapsed_time(e) * 1e3 for s, e in durs)
print(f"overlapped: {wall * 1e6:.0f} us per step ({1 / wall:.0f} it/s); upload under load "
      f"median {d[len(d) // 2]:.0f} us, max {d[-1]:.0f} us")
