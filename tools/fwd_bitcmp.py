"""Dump (mode "save") or compare (mode "cmp") one forward's outputs and the
splat-wise backward's rows at the bench workload, early and after training:
used to check that a forward-kernel variant is bit-identical.
    python tools/fwd_bitcmp.py save|cmp path.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

mode, path = sys.argv[1], sys.argv[2]
cam = survey_camera(1200, 680)
opts = ss.RasterOpts(sh_degree=0)
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(300000, 100)), cam, opts).image
g = ss.GaussianMap.from_scene(survey_scene(300000, 0))
eng = ss.MappingEngine(g, 1200, 680, opts)
eng.fit_capacity(cam)
res = {}


def record(phase, gm):
    out = ss.rasterize_forward(gm, cam, opts)
    gen = torch.Generator("cuda").manual_seed(1)
    gi = torch.randn(out.image.shape, device="cuda", generator=gen)
    g2d = ss.screen_space_grads(out, gi)
    for k in ("image", "final_t", "n_contrib", "k_eff_tiles"):
        res[f"{phase}_{k}"] = getattr(out, k).cpu().numpy()
    res[f"{phase}_g2d"] = g2d.cpu().numpy()


# the same two maps in both processes: the initial one, and (trained here in
# "save" mode, loaded in "cmp" mode) one after 200 training iterations
record("early", g)
if mode == "save":
    for _ in range(200):
        eng.step(cam, tgt)
    eng.synchronize()
    h = eng.gmap.to_numpy()
    for k, v in h.items():
        res[f"map_{k}"] = v
    trained = eng.gmap
else:
    ref0 = np.load(path)
    trained = ss.GaussianMap.from_arrays(ref0["map_positions"], ref0["map_rotations"],
                                         ref0["map_log_scales"], ref0["map_opacity_logits"],
                                         ref0["map_sh"])
record("conv", trained)
if mode == "save":
    np.savez(path, **res)
    print("saved", path)
else:
    ref = np.load(path)
    bad = 0
    for k, v in res.items():
        if k.startswith("map_"):
            continue
        if k.endswith("g2d"):
            sc = np.abs(ref[k]).max(axis=0) + 1e-30
            d = float((np.abs(v - ref[k]) / sc).max())
            print(k, "max rel-to-column-max diff", d)
            bad += d > 1e-5
        else:
            eq = np.array_equal(v, ref[k])
            print(k, "bit-identical" if eq else "DIFFERS", int((v != ref[k]).sum()))
            bad += not eq
    print("RESULT", "OK" if bad == 0 else "MISMATCH")
