"""Per-CTA phase timeline of the binning front end (diagnostics).

Needs the library built with -DSS_FE_TRACE, e.g. on the GPU box:
    make -C paper_2410_00486_b200/csrc clean
    make -C paper_2410_00486_b200/csrc EXTRA=-DSS_FE_TRACE
    python tools/trace_front.py
Stamps (globaltimer, per CTA): 0 start, 1+2p / 2+2p depth pass p before /
after its second grid barrier; direct emission: 10/11 around the chunk-sum
barrier, 12 count walk done, 13 warp prefix done, 14/15 around the count
barrier, 16/17 around the column-prefix barrier, 18 tile starts done, 19
rank walk done; 20+p after depth pass p's first barrier; 24+4p column
histograms loaded, 25+4p local reorder done, 26+4p scatter done (before the
pass's second barrier).  The buffer is cleared (zeros read back first) so
stale stamps of skipped passes do not show."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2410_00486_b200 as ss  # noqa: E402
from paper_2410_00486_b200 import _lib  # noqa: E402
from paper_2410_00486_b200.scene import survey_camera, survey_scene  # noqa: E402

n = int(os.environ.get("PROF_N", 300000))
W = int(os.environ.get("PROF_W", 1200))
H = int(os.environ.get("PROF_H", 680))
g = ss.GaussianMap.from_scene(survey_scene(n, 0))
cam = survey_camera(W, H)
opts = ss.RasterOpts(sh_degree=0)
tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(n, 100)), cam, opts).image
eng = ss.MappingEngine(g, W, H, opts)
eng.fit_capacity(cam)
for _ in range(5):
    eng.step(cam, tgt)
eng.synchronize()
L = _lib.lib()
fn = L.ss_debug_fe_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
clr = L.ss_debug_fe_trace_clear
S = 40
assert clr() == 0
eng.step(cam, tgt)
eng.synchronize()
buf = np.zeros(160 * S, np.uint64)
assert fn(buf.ctypes.data, buf.nbytes) == 0
tr = buf.reshape(160, S).astype(np.int64)
used = tr[:, 0] > 0
tr = tr[used]
base = tr[:, 0].min()
print(f"CTAs {len(tr)}")
for k in range(1, S):
    col = tr[:, k]
    if (col == 0).all():
        continue
    ok = col > 0
    rel = (col[ok] - base) / 1e3
    print(f"stamp {k:2d}: median {np.median(rel):8.2f} us  min {rel.min():8.2f}  max {rel.max():8.2f}")
