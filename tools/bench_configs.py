"""Mapping iterations/s at the SURVEY.md 8.0 configs beyond the headline one
(bench.py measures configs[1]): TUM-shaped S(150k, 640x480), the large
S(1M, 1200x680) per view, and SH3 S(500k, 1200x680).  Device time of K
CUDA-graph steps bracketed by events, L2 flushed between steps.

    python tools/bench_configs.py > profiles/r01_configs.jsonl
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

CONFIGS = [("tum", 150_000, 640, 480, 0), ("replica", 300_000, 1200, 680, 0),
           ("large_per_view", 1_000_000, 1200, 680, 0), ("sh3", 500_000, 1200, 680, 3)]


def main(steps=20, warmup=5):
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for name, n, w, h, deg in CONFIGS:
        opts = ss.RasterOpts(sh_degree=deg)
        cam = survey_camera(w, h)
        tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam,
                                   opts).image.clone()
        eng = ss.MappingEngine(ss.GaussianMap.from_scene(survey_scene(n, 0)), w, h, opts)
        eng.fit_capacity(cam)
        eng.enable_graph()
        for _ in range(warmup):
            eng.step(cam, tgt)
        eng.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        for a, b in ev:
            flush.fill_(0.0)
            a.record()
            eng.step(cam, tgt)
            b.record()
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / steps
        eng.synchronize()
        print(json.dumps({"config": name, "gaussians": n, "image": [w, h], "sh_degree": deg,
                          "it_per_s": 1000.0 / ms, "ms_per_step": ms,
                          "pairs": eng.last_pair_count(), "steps": steps, "warmup": warmup,
                          "dtype": "f32", "data": "synthetic survey scene (SURVEY.md 8d)"}),
              flush=True)
        del eng


if __name__ == "__main__":
    main()
