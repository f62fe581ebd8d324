"""Splat-wise vs pixel-wise backward on B200 (the paper's ablation, PAPER.md
Sec. 3 / Fig. "total iteration": splat-wise backprop gives ~3x the mapping
iterations of pixel-wise backprop).

Both kernels get the same render (forward with checkpoints) and the same
loss gradient (compute_losses of the render against the survey target);
each is timed alone with CUDA events on the launching stream, L2 flushed
between repetitions.  Also reports the whole fused iteration time and the
iteration time with the pixel-wise kernel substituted.

    python tools/ablation_backward.py [--reps 20] > profiles/r01_ablation_backward.jsonl
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

CONFIGS = {"replica": (300_000, 1200, 680), "tum": (150_000, 640, 480)}


def timed(fn, reps, flush):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for a, b in ev:
        flush.fill_(1.0)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return ms[len(ms) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--configs", default="replica,tum")
    ap.add_argument("--train-steps", type=int, default=0,
                    help="fused training steps on the target before timing (converged regime)")
    args = ap.parse_args()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    opts = ss.RasterOpts(sh_degree=0)
    for name in args.configs.split(","):
        n, w, h = CONFIGS[name]
        cam = survey_camera(w, h)
        gmap = ss.GaussianMap.from_scene(survey_scene(n, 0))
        tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam,
                                   opts).image.clone()
        if args.train_steps:
            trainer = ss.MappingEngine(gmap, w, h, opts)
            trainer.fit_capacity(cam)
            trainer.enable_graph()
            for _ in range(args.train_steps):
                trainer.step(cam, tgt)
            trainer.synchronize()
            gmap = trainer.gmap
        out = ss.rasterize_forward(gmap, cam, opts)
        lb = ss.compute_losses(out.image, tgt, gmap.opacity_logits)
        g = lb.grad_image
        splat_ms = timed(lambda: ss.screen_space_grads(out, g), args.reps, flush)
        pixel_ms = timed(lambda: ss.screen_space_grads_pixelwise(out, g), args.reps, flush)
        a = ss.screen_space_grads(out, g).double()
        b = ss.screen_space_grads_pixelwise(out, g).double()
        agree = float((a - b).norm() / a.norm())
        # whole fused iteration (CUDA graph), and with the pixel-wise kernel swapped in
        eng = ss.MappingEngine(gmap.clone(), w, h, opts)
        eng.fit_capacity(cam)
        eng.enable_graph()
        it_ms = timed(lambda: eng.step(cam, tgt), args.reps, flush)
        eng.synchronize()
        line = {
            "config": {"workload": f"S({n},{w}x{h}) SH0, one view"
                                   + (f", after {args.train_steps} training steps"
                                      if args.train_steps else ""),
                       "gaussians": n, "image": [w, h], "pairs": out.pair_count},
            "backward_splatwise_ms": splat_ms,
            "backward_pixelwise_ms": pixel_ms,
            "speedup_splat_over_pixel": pixel_ms / splat_ms,
            "g2d_normwise_diff": agree,
            "iteration_ms_splatwise": it_ms,
            "iteration_ms_pixelwise": it_ms - splat_ms + pixel_ms,
            "iterations_ratio": (it_ms - splat_ms + pixel_ms) / it_ms,
            "note": "backward kernels timed alone (median of reps, L2 flushed); the "
                    "pixel-wise iteration substitutes its kernel time in the fused step",
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
