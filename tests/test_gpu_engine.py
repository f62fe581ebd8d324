"""MappingEngine behaviour on the GPU: graph captures across densify, error
handling before the update (api.py:74-79, optimizer.py:111-113), capacity
fitting, one graph for every keyframe target, the keyframe batch against the
oracle's sum over views, and the keyframe-sharded step with
two ranks (world 2 over gloo on one GPU: host-side collective, no kernel of
one rank waits on the other's)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle as orc  # noqa: E402
from helpers import fixture_camera, fixture_scene, load, normwise  # noqa: E402


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _small(n=3000, w=96, h=72, seed=4, views=1):
    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    opts = ss.RasterOpts(sh_degree=0)
    cams = [survey_camera(w, h, v, views) for v in range(views)]
    tm = ss.GaussianMap.from_scene(survey_scene(n, seed + 100))
    tg = [ss.rasterize_forward(tm, c, opts).image.clone() for c in cams]
    return ss, survey_scene(n, seed), cams, tg, opts


def _params(g):
    return {f: getattr(g, f).detach().cpu().numpy().copy()
            for f in ("positions", "rotations", "log_scales", "opacity_logits", "sh_dc",
                      "grad2d_accum", "obs_count")}


def test_graph_dropped_when_densify_keeps_the_count():
    """a densify that leaves N unchanged still installs new map
    and moment tensors; the captured graph must not replay into the old
    ones.  Graph engine == stream engine through the densify."""
    _need_gpu()
    ss, sc, cams, tg, opts = _small()
    # thresholds no Gaussian crosses: nothing cloned, split or pruned
    cfg = ss.EngineConfig(densify=ss.DensifyConfig(interval=3, grad_threshold=1e9,
                                                   prune_opacity=1e-9))
    ga, gb = ss.GaussianMap.from_scene(sc), ss.GaussianMap.from_scene(sc)
    ea = ss.MappingEngine(ga, 96, 72, opts, cfg)
    eb = ss.MappingEngine(gb, 96, 72, opts, cfg)
    eb.enable_graph()
    for _ in range(7):  # densify runs before steps 4 and 7
        ea.step(cams[0], tg[0])
        eb.step(cams[0], tg[0])
    ea.synchronize()
    eb.synchronize()
    assert len(ga) == len(gb) == len(sc.positions)
    lr = dict(positions=1.6e-4, rotations=1e-3, log_scales=5e-3, opacity_logits=5e-2,
              sh_dc=2.5e-3)
    pa, pb = _params(ga), _params(gb)
    for f, r in lr.items():
        d = np.abs(pa[f] - pb[f])
        # float-atomic g2d rows: runs agree to rounding; Adam bounds sign flips
        assert d.max() <= 14 * r + 1e-5, f
        assert (d > 1e-3 * r + 1e-6).mean() < 0.03, f
    # the stale-graph failure mode: the graph engine's map stops moving
    assert np.abs(pb["positions"] - sc.positions.astype(np.float32)).max() > 1e-4


def test_one_graph_serves_every_keyframe_target():
    _need_gpu()
    ss, sc, cams, tg, opts = _small(views=3)
    g = ss.GaussianMap.from_scene(sc)
    eng = ss.MappingEngine(g, 96, 72, opts)
    eng.fit_capacity(cams)
    eng.enable_graph()
    gs = ss.GaussianMap.from_scene(sc)
    es = ss.MappingEngine(gs, 96, 72, opts)
    es.fit_capacity(cams)
    for k in range(6):
        eng.step(cams[k % 3], tg[k % 3])
        es.step(cams[k % 3], tg[k % 3])
    eng.synchronize()
    es.synchronize()
    assert len(eng._graphs) == 1
    la, lb = eng.losses(), es.losses()
    np.testing.assert_allclose([x[1] for x in la], [x[1] for x in lb], rtol=1e-5)


def test_fit_capacity_only_grows():
    _need_gpu()
    ss, sc, cams, tg, opts = _small(views=4)
    eng = ss.MappingEngine(ss.GaussianMap.from_scene(sc), 96, 72, opts, pair_capacity=64)
    pmax = eng.fit_capacity(cams)
    cap = eng.pair_capacity
    assert cap >= pmax
    p0 = eng.fit_capacity(cams[0], margin=1.0)
    assert p0 <= pmax and eng.pair_capacity == cap


def test_nonfinite_gradient_raises_and_leaves_map_unchanged():
    """A NaN target makes every pixel gradient non-finite, so every Gaussian
    that blended gets a non-finite gradient: the fused chain+Adam leaves
    those Gaussians untouched (parameters, moments, statistics) and the
    engine raises FloatingPointError when the step's status arrives."""
    _need_gpu()
    ss, sc, cams, tg, opts = _small()
    g = ss.GaussianMap.from_scene(sc)
    seen = ss.rasterize_forward(g, cams[0], opts).contributed.cpu().numpy()
    assert seen.sum() > 100
    before = _params(g)
    eng = ss.MappingEngine(g, 96, 72, opts)
    bad = torch.full_like(tg[0], float("nan"))
    eng.step(cams[0], bad)
    with pytest.raises(FloatingPointError):
        eng.synchronize()
    after = _params(g)
    for f in before:
        np.testing.assert_array_equal(after[f][seen], before[f][seen], err_msg=f)
    for k in ("position", "rotation", "opacity_logit"):
        assert np.all(eng.state.m[k].cpu().numpy()[seen] == 0.0), k


def test_zero_quaternion_raises():
    _need_gpu()
    ss, sc, cams, tg, opts = _small()
    sc.rotations[7] = 0.0
    eng = ss.MappingEngine(ss.GaussianMap.from_scene(sc), 96, 72, opts)
    eng.step(cams[0], tg[0])
    with pytest.raises(ValueError, match="zero-norm quaternion"):
        eng.synchronize()


def test_multiview_raises_before_adam_on_bad_parameter():
    """the keyframe batch checks the error words (one host read
    after the views) before Adam touches the map."""
    _need_gpu()
    ss, sc, cams, tg, opts = _small(views=2)
    sc.positions[11, 0] = np.inf
    g = ss.GaussianMap.from_scene(sc)
    before = _params(g)
    eng = ss.MappingEngine(g, 96, 72, opts)
    with pytest.raises(ValueError, match="non-finite parameter in primitive 11"):
        eng.multiview_step(cams, tg)
    after = _params(g)
    for f in before:
        np.testing.assert_array_equal(after[f], before[f], err_msg=f)


def _f32_omap(sc):
    f = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    return orc.OMap(f(sc.positions), f(sc.rotations), f(sc.log_scales), f(sc.opacity_logits),
                    f(sc.sh))


def test_multiview_batch_equals_oracle_sum_over_views():
    """A17 against the oracle: the engine's flat buffer after the views
    (every plane) == sum over views of the oracle's per-view ParamGrads of
    the same float32 map (trainer.py:194-207 per view), the regulariser
    gradient once; the statistics planes == per-view accumulate_grad_stats."""
    _need_gpu()
    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.distributed import flat_layout
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    n, w, h, V = 3000, 96, 64, 3
    sc, tsc = survey_scene(n, 5), survey_scene(n, 105)
    cams = [survey_camera(w, h, v, V) for v in range(V)]
    tm = orc.OMap(tsc.positions, tsc.rotations, tsc.log_scales, tsc.opacity_logits, tsc.sh)
    tg_np = [orc.rasterize(tm, c, sh_degree=0, with_checkpoints=False).image for c in cams]
    tg = [torch.as_tensor(t, dtype=torch.float32, device="cuda") for t in tg_np]
    gm = ss.GaussianMap.from_scene(sc)
    eng = ss.MappingEngine(gm, w, h, ss.RasterOpts(sh_degree=0))
    captured = {}
    eng.multiview_step(cams, tg, allreduce=lambda f: captured.setdefault("flat", f.clone()))
    flat = captured["flat"].cpu().numpy().astype(np.float64)
    om = _f32_omap(sc)
    total, lbs = orc.multiview_grads(om, cams, [t.astype(np.float32).astype(np.float64)
                                                for t in tg_np], sh_degree=0)
    layout, size = flat_layout(n, 0)
    assert flat.shape[0] == size and flat[-2:].tolist() == [0.0, 0.0]
    v = {name: flat[off:off + k * n] for name, k, off in layout}
    for name, ref in (("position", total.position), ("rotation", total.rotation),
                      ("log_scale", total.log_scale), ("opacity", total.opacity_logit),
                      ("sh_dc", total.sh[:, 0, :]), ("pos2d", total.pos2d_grad_norm)):
        assert normwise(v[name], ref.reshape(-1)) <= 1e-3, name
    # statistics increments: per-view accumulate_grad_stats
    ref_map = _f32_omap(sc)
    for c, t in zip(cams, tg_np):
        r = orc.rasterize(om, c, sh_degree=0)
        lb = orc.losses(r.image, t.astype(np.float32).astype(np.float64), om.opacity_logits)
        gv = orc.chain(om, c, r.proj, orc.backward_splat(r, lb.grad_image), r.contributed)
        orc.accumulate_grad_stats(ref_map, gv)
    np.testing.assert_array_equal(v["stat_cnt"].astype(np.int64), ref_map.obs_count)
    assert normwise(v["stat_g2d"], ref_map.grad2d_accum) <= 1e-3
    assert normwise(v["stat_g3d"], ref_map.grad3d_accum.reshape(-1)) <= 1e-3
    np.testing.assert_array_equal(gm.obs_count.cpu().numpy(), ref_map.obs_count)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.distributed import ShardedMapper, replica_checksum
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    n, w, h, V = 3000, 96, 64, 4
    opts = ss.RasterOpts(sh_degree=0)
    cams = [survey_camera(w, h, v, V) for v in range(V)]
    tm = ss.GaussianMap.from_scene(survey_scene(n, 106))
    tg = [ss.rasterize_forward(tm, c, opts).image.clone() for c in cams]
    g = ss.GaussianMap.from_scene(survey_scene(n, 6))
    eng = ss.MappingEngine(g, w, h, opts, pair_capacity=64)  # forces the redo path once
    sm = ShardedMapper(eng)
    flats = []
    orig = eng.multiview_step

    def spy(*a, **k):
        ar = k["allreduce"]
        k["allreduce"] = lambda f: (ar(f), flats.append(f.clone()))
        return orig(*a, **k)
    eng.multiview_step = spy
    for _ in range(3):
        sm.step(cams, tg)
    eng.synchronize()
    arrays = [getattr(g, f) for f in ("positions", "rotations", "log_scales", "opacity_logits",
                                      "sh_dc", "grad2d_accum", "grad3d_accum", "obs_count")]
    out_q.put((rank, replica_checksum(arrays), [f.cpu().numpy() for f in flats],
               {f: getattr(g, f).cpu().numpy() for f in ("positions", "obs_count")}))
    dist.destroy_process_group()


def test_sharded_mapper_two_ranks_equals_one_rank_batch():
    """The CUDA engine's keyframe-sharded step, world 2 (views 0,2 | 1,3),
    vs one process running the whole 4-view batch: the reduced gradient
    buffers agree to float rounding, obs_count exactly, and the two ranks'
    replicas are byte-identical after 3 steps (one of them redone after a
    pair overflow on both ranks)."""
    _need_gpu()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1]  # replicas byte-identical
    # single-process reference of the same batch
    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    n, w, h, V = 3000, 96, 64, 4
    opts = ss.RasterOpts(sh_degree=0)
    cams = [survey_camera(w, h, v, V) for v in range(V)]
    tm = ss.GaussianMap.from_scene(survey_scene(n, 106))
    tg = [ss.rasterize_forward(tm, c, opts).image.clone() for c in cams]
    g = ss.GaussianMap.from_scene(survey_scene(n, 6))
    eng = ss.MappingEngine(g, w, h, opts)
    eng.fit_capacity(cams)
    flats = []
    for _ in range(3):
        eng.multiview_step(cams, tg, allreduce=lambda f: flats.append(f.clone()))
    eng.synchronize()
    # the two-rank run overflowed its 64-pair buffers on the first pass: that
    # pass's flags tail reads (2, 0) on every rank and the step was redone
    assert res[0][2][0][-2] == 2.0
    done = [f for f in res[0][2] if f[-2] == 0.0]
    assert len(done) == 3 and len(flats) == 3
    for a, b in zip(done, flats):
        assert normwise(a, b.cpu().numpy()) <= 1e-5
    np.testing.assert_array_equal(res[0][3]["obs_count"], g.obs_count.cpu().numpy())
    d = np.abs(res[0][3]["positions"] - g.positions.cpu().numpy())
    assert d.max() <= 6 * 1.6e-4 and (d > 1e-6).mean() < 0.02


def test_scheduled_mapper_matches_oracle_trainer_selection():
    """F1 with the real engine: ScheduledMapper(synchronous=True) picks the
    same keyframe sequence as the reference trainer loop (trainer.py:194-210:
    select -> train_one -> record_result(total loss)) run on the oracle with
    the same scheduler (pinned to the reference's traces in
    tests/test_scheduler.py), and records matching losses."""
    _need_gpu()
    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    n, w, h, K, iters = 2000, 64, 48, 6, 40
    sc, tsc = survey_scene(n, 8), survey_scene(n, 108)
    cams = [survey_camera(w, h, v, K) for v in range(K)]
    tm = orc.OMap(tsc.positions, tsc.rotations, tsc.log_scales, tsc.opacity_logits, tsc.sh)
    tg_np = [orc.rasterize(tm, c, sh_degree=0, with_checkpoints=False).image
             .astype(np.float32).astype(np.float64) for c in cams]
    # the oracle trainer
    om = _f32_omap(sc)
    st = orc.OAdam.for_map(om)
    sch = ss.KeyframeScheduler(d=2, r0=2, seed=5)
    for k in range(K):
        sch.add_keyframe(k)
    ref_picks, ref_loss = [], {}
    for _ in range(iters):
        kf = sch.select()
        lb = orc.iteration(om, cams[kf], tg_np[kf], st, sh_degree=0)
        sch.record_result(kf, lb.total)
        ref_picks.append(kf)
        ref_loss[kf] = lb.total
    # the engine
    eng = ss.MappingEngine(ss.GaussianMap.from_scene(sc), w, h, ss.RasterOpts(sh_degree=0))
    eng.fit_capacity(cams)
    eng.enable_graph()
    sm = ss.ScheduledMapper(eng, ss.KeyframeScheduler(d=2, r0=2, seed=5), synchronous=True)
    for k in range(K):
        sm.add_keyframe(k, cams[k], torch.as_tensor(tg_np[k], dtype=torch.float32,
                                                    device="cuda"))
    picks = [sm.step() for _ in range(iters)]
    sm.synchronize()
    assert picks == ref_picks
    assert sm.sched.remaining == sch.remaining
    for k, v in ref_loss.items():
        assert abs(sm.kf_loss[k] - v) <= 1e-3 * abs(v), (k, sm.kf_loss[k], v)
    assert len(eng._graphs) == 1



def test_upload_target_chunked_copy_and_errors():
    """MappingEngine.upload_target: the row chunks copied on concurrent copy
    streams reassemble the keyframe exactly in the requested slot, ordered
    after `after`; a step fed the slot matches a step fed the same target
    through step()'s own staging copy; wrong dtype / shape / unpinned host
    memory are rejected."""
    _need_gpu()
    import paper_2410_00486_b200 as ss
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    cam = survey_camera(160, 120)
    opts = ss.RasterOpts(sh_degree=0)
    tgt = ss.rasterize_forward(ss.GaussianMap.from_scene(survey_scene(4000, 71)), cam,
                               opts).image
    host = tgt.cpu().pin_memory()
    e1 = ss.MappingEngine(ss.GaussianMap.from_scene(survey_scene(4000, 72)), 160, 120, opts)
    e2 = ss.MappingEngine(ss.GaussianMap.from_scene(survey_scene(4000, 72)), 160, 120, opts)
    for k in (1, 3, 4):
        before = torch.cuda.Event()
        before.record()
        ev = e1.upload_target(host, 1, after=before, chunks=k)
        torch.cuda.current_stream().wait_event(ev)
        assert torch.equal(e1.target_buffer(slot=1), tgt), k
    for _ in range(3):
        ev = e1.upload_target(host, 1)
        torch.cuda.current_stream().wait_event(ev)
        e1.step(cam, e1.target_buffer(slot=1))
        e2.step(cam, tgt)
    e1.synchronize()
    e2.synchronize()
    # (the backward's per-tile red.add rows sum in any order: last-bit noise)
    assert torch.allclose(e1.gmap.positions, e2.gmap.positions, rtol=0, atol=1e-5)
    with pytest.raises(ValueError):
        e1.upload_target(host.double().pin_memory(), 0)
    with pytest.raises(ValueError):
        e1.upload_target(tgt.cpu(), 0)
    with pytest.raises(ValueError):
        e1.upload_target(host[:-1].clone().pin_memory(), 0)
