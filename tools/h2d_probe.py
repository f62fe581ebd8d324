"""Pinned host -> device copy rate of one keyframe (9.8 MB) on this box: one
copy vs the same bytes split over several streams (copy engines)."""
import time

import torch

n = 1200 * 680 * 3
x = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for k in (1, 2, 4):
    chunks = [(i * n // k, (i + 1) * n // k) for i in range(k)]
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(20):
            for (a, b), s in zip(chunks, streams):
                with torch.cuda.stream(s):
                    d[a:b].copy_(x[a:b], non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 20
    print(f"{k} stream(s): {dt * 1e3:.3f} ms per 9.8 MB = {n * 4 / dt / 1e9:.1f} GB/s")
