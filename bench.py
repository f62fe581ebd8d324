"""Benchmark: mapping iterations/sec (fwd + splat-wise bwd + Adam) at
1200x680 with 300k Gaussians (BASELINE.json metric, configs[1]).

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]

One process per GPU (torchrun for N > 1, NCCL).  N = 1: the fused single-
view iteration (MappingEngine.step).  N > 1: keyframe sharding -- every
rank renders and back-propagates its own view of the replicated map, the
flat per-Gaussian gradient buffer is summed with one NCCL all-reduce, and
every rank applies the identical Adam step (weak scaling: one view per
GPU per step; value = views * steps / time, all ranks).

``--impl reference`` times the reference's CPU implementation of the path
as restated in oracle/ (float64, all host threads; the reference itself is
Python + numba and cannot travel to the GPU box) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "mapping iters/sec (fwd+bwd+Adam) at 1200×680, 300k Gaussians; HBM GB/s"
WORKLOAD = dict(n=300_000, width=1200, height=680, sh_degree=0)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=WORKLOAD["n"])
    ap.add_argument("--width", type=int, default=WORKLOAD["width"])
    ap.add_argument("--height", type=int, default=WORKLOAD["height"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=25.0)
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ algorithmic bytes
def algorithmic_bytes(n, m, p, hw, t, c, e, u=None, G=14):
    """SURVEY.md 8d per-stage compulsory HBM traffic (float32, int32 ids,
    u64 keys, sort = one read + one write), bytes per iteration.  c =
    checkpoint slots (32-position buckets, sum ceil(k_eff/32)): the forward
    writes a (T, rgb) state and a blend mask per pixel per slot; u = backward
    work units (64 positions = 2 slots), each reading one state slot and two
    mask slots."""
    u = c / 2 if u is None else u
    st = {
        "preprocess": n * G * 4 + n * 48,
        "scan": n * 8,
        "dup": n * 20 + p * 12,
        "sort": p * 24,
        "ranges": p * 8 + t * 8,
        "blend_forward": p * 4 + m * 36 + hw * 20 + c * (4096 + 1024) + n,
        "loss": hw * 36,
        "backward": e * 4 + m * 36 + u * (4096 + 2048) + hw * 28 + m * 36,
        "chain": m * 36 + n * G * 8 + n * 5,
        "adam": n * G * 28,
        "stats": n * 57,
    }
    return st


def ncu_stats(kernel):
    """Per-launch figures of `kernel` from the committed ncu --set full
    capture summary (profiles/ncu_traffic.json), else {}."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(kernel) or {}
    except Exception:
        return {}


def ncu_traffic(kernel):
    """dram read+write bytes per launch of `kernel` (ncu), else None."""
    return ncu_stats(kernel).get("dram_bytes")


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------- CPU oracle
def cpu_iteration_setup(args):
    import numpy as np

    import oracle as orc
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    sc = survey_scene(args.n, 0)
    cam = survey_camera(args.width, args.height)
    om = orc.OMap(sc.positions, sc.rotations, sc.log_scales, sc.opacity_logits, sc.sh)
    return orc, om, cam, np


def cpu_target(args, orc, cam):
    from paper_2410_00486_b200.scene import survey_scene
    tsc = survey_scene(args.n, 100)
    tm = orc.OMap(tsc.positions, tsc.rotations, tsc.log_scales, tsc.opacity_logits, tsc.sh)
    return orc.rasterize(tm, cam, sh_degree=0, with_checkpoints=False).image


def run_cpu_iterations(args, max_iters, budget_s):
    """Oracle train_one sequence (trainer.py:199-208) in float64, all threads."""
    orc, om, cam, np = cpu_iteration_setup(args)
    threads = os.cpu_count() or 1
    orc.set_threads(threads)
    target = cpu_target(args, orc, cam)
    st = orc.OAdam.for_map(om)
    times = []
    t_all = time.perf_counter()
    while len(times) < max_iters:
        t0 = time.perf_counter()
        orc.iteration(om, cam, target, st, sh_degree=0)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s:
            break
    return times, threads


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    import platform
    warm = min(args.warmup, 1)
    times, threads = run_cpu_iterations(args, warm + args.steps, budget_s=150.0)
    timed = times[warm:] if len(times) > warm else times
    it_s = len(timed) / sum(timed)
    line = {
        "impl": "reference", "metric": METRIC, "value": it_s, "unit": "it/s",
        "n_gpus": args.gpus, "steps": len(timed), "warmup": warm,
        "ms_per_step": 1000.0 * sum(timed) / len(timed), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"replica-shaped S({args.n},{args.width}x{args.height}) SH0 "
                               "single view (BASELINE configs[1])", "gaussians": args.n,
                   "image": [args.width, args.height], "sh_degree": 0},
        "cpu_baseline": {"value": it_s, "unit": "it/s", "cores": threads, "kind": "port",
                         "sample": f"{len(timed)} full float64 iterations of the oracle "
                                   f"restatement (oracle/, {threads} OpenMP threads, "
                                   f"host {platform.processor() or platform.machine()}); "
                                   f"requested {args.steps}, capped at 150 s"},
        "e2e": {"value": it_s, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU arm
def main():
    args = _args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.scene import survey_camera, survey_scene

    W, H, N = args.width, args.height, args.n
    sc = survey_scene(N, 0)
    opts = ss.RasterOpts(sh_degree=0)
    gmap = ss.GaussianMap.from_scene(sc)
    views = max(world, 1)
    cams = [survey_camera(W, H, v, views) for v in range(views)]
    # targets: render of S(N, seed+100) from each view (rendered
    # on the GPU here -- the oracle takes seconds per 300k render)
    tmap = ss.GaussianMap.from_scene(survey_scene(N, 100))
    targets = [ss.rasterize_forward(tmap, c, opts).image.clone() for c in cams]
    del tmap
    eng = ss.MappingEngine(gmap, W, H, opts)
    pcount = eng.fit_capacity(cams[rank % views])
    if world == 1:
        eng.enable_graph()  # the whole iteration is replayed as one CUDA graph
    my_cam, my_tgt = cams[rank % views], targets[rank % views]
    # the device-timed steps read the target from the engine's own buffer (the
    # one its captured graph reads); the e2e run below passes host-uploaded
    # buffers, which step() copies there
    eng.target_buffer().copy_(my_tgt)

    from paper_2410_00486_b200.distributed import ShardedMapper
    sharded = ShardedMapper(eng, rank, world) if world > 1 else None

    def one_step():
        if sharded is not None:
            sharded.step(cams, targets)  # one view per rank, one NCCL all-reduce
        else:
            eng.step(my_cam, eng.target_buffer())

    # L2 flush buffer (> 126 MB L2), written between timed steps
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(max(args.warmup, 3)):
        one_step()
    eng.synchronize() if world == 1 else torch.cuda.synchronize()

    # parameters + Adam state after warm-up: the e2e run below restores them
    # in place (graph pointers stay valid) so it times the same iterations
    # as the device-timed run -- the per-iteration cost drifts as training
    # lowers opacities (profiles/r01_training_drift.txt)
    snap = None
    if world == 1:
        snap = ([getattr(eng.gmap, f).clone() for f in eng.gmap.FIELDS],
                {k: t.clone() for k, t in eng.state.m.items()},
                {k: t.clone() for k, t in eng.state.v.items()}, eng.state.step_count)

    # ---- timed region: per-step CUDA events, L2 flushed between steps
    sampler = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    launches0 = eng.launches
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.fill_(float(k))
        starts[k].record()
        one_step()
        ends[k].record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world == 1:
        eng.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    launches = eng.launches - launches0
    if dist is not None:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = views * args.steps / (total_ms / 1000.0)

    # ---- per-kernel timing (instrumented steps, outside the timed region)
    eng.profile = []
    prof_steps = 5
    for _ in range(prof_steps):
        one_step()
    torch.cuda.synchronize()
    stages = {}
    prof = eng.profile
    eng.profile = None
    for (a, ea), (b, eb) in zip(prof[:-1], prof[1:]):
        if b == "begin":
            continue
        stages.setdefault(b, []).append(ea.elapsed_time(eb))
    stage_ms = {k: sum(v) / len(v) for k, v in stages.items()}

    # ---- workload statistics for the algorithmic-byte model
    st = eng.status.cpu().numpy()
    P = int(st[3])
    U = int(st[5])  # backward work units (64 list positions)
    M = int(st[6])
    E = int(eng.k_eff.sum().item())
    C = int(((eng.k_eff.long() + 31) // 32).sum().item())  # checkpoint slots
    HW = W * H
    T = eng.n_tiles
    algo = algorithmic_bytes(N, M, P, HW, T, C, E, U)
    peak, peak_src = load_peaks()
    per_kernel = {
        "blend_forward": algo["blend_forward"],
        "backward": algo["backward"],
        "binning": algo["scan"] + algo["dup"] + algo["sort"] + algo["ranges"],
        "loss": algo["loss"],
        "chain_adam": algo["chain"] + algo["adam"] + algo["stats"],
        "preprocess": algo["preprocess"],
    }
    dom = max((k for k in stage_ms if k in per_kernel), key=lambda k: stage_ms[k])
    ach = per_kernel[dom] / (stage_ms[dom] / 1000.0) / 1e9
    it_bytes = sum(algo.values())

    # ---- end to end through the public API with host buffers (N=1): every
    # step uploads its keyframe target from pinned host memory (on a copy
    # stream, double-buffered so the upload of step k+1 overlaps step k) and
    # the step's loss/status snapshot comes back to the host
    e2e = None
    if world == 1 and not args.no_e2e:
        eng.synchronize()
        for f, t in zip(eng.gmap.FIELDS, snap[0]):
            getattr(eng.gmap, f).copy_(t)
        for k, t in snap[1].items():
            eng.state.m[k].copy_(t)
        for k, t in snap[2].items():
            eng.state.v[k].copy_(t)
        eng.state.step_count = snap[3]
        host_tgt = my_tgt.cpu().pin_memory()
        bufs = [torch.empty_like(my_tgt), torch.empty_like(my_tgt)]
        copy_stream = torch.cuda.Stream()
        uploaded = [torch.cuda.Event(), torch.cuda.Event()]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]
        main = torch.cuda.current_stream()

        def upload(k):
            b = k % 2
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(consumed[b])
                bufs[b].copy_(host_tgt, non_blocking=True)
                uploaded[b].record(copy_stream)

        def e2e_step(k):
            b = k % 2
            main.wait_event(uploaded[b])
            eng.step(my_cam, bufs[b])
            consumed[b].record(main)
            upload(k + 2)

        for b in range(2):
            consumed[b].record(main)
        upload(0)
        upload(1)
        for k in range(2):  # capture the graphs of both input buffers
            e2e_step(k)
        eng.synchronize()
        torch.cuda.synchronize()
        # the same number of iterations as the device-timed run, from the
        # same state (the 2 graph-capture steps above are not timed)
        n_e2e = args.steps
        t0 = time.perf_counter()
        for k in range(2, 2 + n_e2e):
            e2e_step(k)
        eng.synchronize()  # every step's loss is on the host
        wall = time.perf_counter() - t0
        e2e = {"value": n_e2e / wall, "unit": "it/s", "steps": n_e2e,
               "h2d_bytes_per_step": int(host_tgt.numel() * 4),
               "d2h_bytes_per_step": int(eng._host.shape[1] * 8),
               "timing": "wall clock over the same iterations as `value` (state restored), "
                         "host pinned target upload per step (copy stream, double-buffered) "
                         "+ per-step loss/status read back"}

    # ---- CPU baseline (rank 0, N = 1): bounded oracle sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import platform
        times, threads = run_cpu_iterations(args, 3, args.cpu_budget_s)
        cpu = {"value": len(times) / sum(times), "unit": "it/s", "cores": threads,
               "kind": "port", "sample": f"{len(times)} full float64 iterations of the oracle "
                                        f"restatement of the reference path (oracle/), same "
                                        f"scene/camera, {threads} OpenMP threads on "
                                        f"{platform.machine()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"replica-shaped S({N},{W}x{H}) SH0, "
                                   f"{'single view' if world == 1 else '1 view per GPU, NCCL all-reduce'}"
                                   " (BASELINE configs[1])", "gaussians": N, "image": [W, H],
                       "sh_degree": 0, "pairs": P, "visible": M, "checkpoint_slots": C,
                       "backward_units": U,
                       "l2": "256 MB buffer written between timed steps (outside the events)",
                       "phase": f"iterations {max(args.warmup, 3) + 1}-"
                                f"{max(args.warmup, 3) + args.steps} from the survey "
                                "initialisation (the cost per iteration rises ~2x by "
                                "iteration 150 as training lowers opacities)",
                       "parallelism": f"keyframe-sharded x{world}" if world > 1 else "single GPU"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak,
                         "unit": "GB/s", "frac": ach / peak, "traffic": ncu_traffic(dom),
                         "algorithmic_bytes": per_kernel[dom], "avg_ms": stage_ms[dom],
                         "peak_source": peak_src,
                         "ncu": {k: v for k, v in ncu_stats(dom).items()
                                 if k in ("issue_slots_pct", "warps_active_pct")},
                         "note": "FP32 CUDA-core kernel bound by instruction issue, "
                                 "FMA-pipe occupancy and dependent latency (ncu: issue "
                                 "slots ~55 %, FMA pipe ~56 %, 4 warps/SMSP at 128 regs), "
                                 "not by HBM; no tensor-core work on this path"},
            "iteration_roofline": {"algorithmic_MB": it_bytes / 1e6,
                                   "achieved_GBs": it_bytes * value / views / 1e9,
                                   "frac": it_bytes * value / views / 1e9 / peak},
            "stage_ms": stage_ms,
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    _ = (np, pcount)
    return 0


if __name__ == "__main__":
    sys.exit(main())
