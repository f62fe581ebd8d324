"""Keyframe-sharded step on CPU: world_size 2 over gloo.

The product's ShardedMapper drives an oracle-backed engine double through
one keyframe-batch step: each rank sums the oracle gradients of its shard
of the views into the product's flat layout (distributed.flat_layout), the
buffers are all-reduced, and every rank applies the same Adam step.
Checks: the reduced buffer equals the single-process sum over all views
(the builder-defined batch oracle, A17), the update equals one oracle
adam_step on that sum, and the replicas are byte-identical afterwards.
The CUDA engine's own multi-rank step is covered on the GPU
(tests/test_gpu_engine.py, world 2 over gloo).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2
N_VIEWS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _flat(g, seen_mask, sh_degree=0):
    """Oracle grads of one view -> the engine's flat buffer, laid out by the
    product's own distributed.flat_layout (the layout MappingEngine uses)."""
    from paper_2410_00486_b200.distributed import flat_layout
    n = len(g)
    seen = seen_mask.astype(np.float64)
    planes = {"position": g.position, "rotation": g.rotation, "log_scale": g.log_scale,
              "opacity": g.opacity_logit, "sh_dc": g.sh[:, 0, :], "sh_rest": g.sh[:, 1:, :],
              "pos2d": g.pos2d_grad_norm, "stat_g2d": g.pos2d_grad_norm * seen,
              "stat_g3d": g.position * seen[:, None], "stat_cnt": seen}
    layout, total = flat_layout(n, sh_degree)
    out = np.zeros(total)
    for name, k, off in layout:
        if k:
            out[off:off + k * n] = np.asarray(planes[name], np.float64).reshape(-1)
    return out


def _unflat(orc, buf, n, sh_degree=0):
    from paper_2410_00486_b200.distributed import flat_layout
    layout, _ = flat_layout(n, sh_degree)
    v = {name: buf[off:off + k * n] for name, k, off in layout}
    sh = np.zeros((n, 16, 3))
    sh[:, 0, :] = v["sh_dc"].reshape(n, 3)
    if sh_degree:
        sh[:, 1:, :] = v["sh_rest"].reshape(n, 15, 3)
    g = orc.OGrads(v["position"].reshape(n, 3), v["rotation"].reshape(n, 4),
                   v["log_scale"].reshape(n, 3), v["opacity"].copy(), sh, v["pos2d"].copy(),
                   v["stat_cnt"] > 0)
    return g, v


def _scene():
    import oracle as orc
    from paper_2410_00486_b200.scene import survey_camera, survey_scene
    sc = survey_scene(600, 4)
    tsc = survey_scene(600, 104)
    cams = [survey_camera(48, 40, v, N_VIEWS) for v in range(N_VIEWS)]
    tm = orc.OMap(tsc.positions, tsc.rotations, tsc.log_scales, tsc.opacity_logits, tsc.sh)
    targets = [orc.rasterize(tm, c, sh_degree=0, with_checkpoints=False).image for c in cams]
    om = orc.OMap(sc.positions, sc.rotations, sc.log_scales, sc.opacity_logits, sc.sh)
    return orc, om, cams, targets


def _view_flat(orc, om, cam, tgt, add_reg):
    r = orc.rasterize(om, cam, sh_degree=0)
    lb = orc.losses(r.image, tgt, om.opacity_logits)
    g = orc.chain(om, cam, r.proj, orc.backward_splat(r, lb.grad_image), r.contributed)
    if add_reg:
        g.opacity_logit = g.opacity_logit + lb.grad_opacity_logit
    return _flat(g, r.contributed), g


class OracleEngine:
    """Test double with MappingEngine.multiview_step's contract, computing
    with the CPU oracle (no GPU here): per-view grads summed into the flat
    buffer (the product's layout), the tail flags, the all-reduce hook, then
    Adam and the statistics update from the reduced buffer -- so the real
    ShardedMapper drives it exactly as it drives the CUDA engine."""

    def __init__(self, orc, om):
        self.orc, self.gmap = orc, om
        self.state = orc.OAdam.for_map(om)
        self.reduced = None

    def multiview_step(self, cams, tgts, tds=None, allreduce=None, add_reg=True):
        orc, om = self.orc, self.gmap
        n = len(om)
        local = _flat(orc.OGrads(np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3)),
                                 np.zeros(n), np.zeros((n, 16, 3)), np.zeros(n),
                                 np.zeros(n, bool)), np.zeros(n, bool))
        for v, (c, t) in enumerate(zip(cams, tgts)):
            local += _view_flat(orc, om, c, t, add_reg=(add_reg and v == 0))[0]
        buf = torch.from_numpy(local).double()
        if allreduce is not None:
            allreduce(buf)
        self.reduced = buf.numpy().copy()
        assert self.reduced[-2:].tolist() == [0.0, 0.0]  # no rank overflowed or failed
        g, v = _unflat(orc, self.reduced, n)
        orc.adam(om, g, self.state)
        seen = v["stat_cnt"] > 0
        om.grad2d_accum += v["stat_g2d"]
        om.grad3d_accum += v["stat_g3d"].reshape(n, 3)
        om.obs_count += v["stat_cnt"].astype(np.int64)
        assert np.all(v["stat_cnt"][~seen] == 0)
        return []


def _worker(rank, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2410_00486_b200.distributed import ShardedMapper, checksums_agree, shard_views
    orc, om, cams, targets = _scene()
    eng = OracleEngine(orc, om.copy())
    sm = ShardedMapper(eng)
    assert (sm.rank, sm.world) == (rank, WORLD)
    sm.step(cams, targets)
    # single-process oracle of the batch (A17): every view's grads summed, the
    # opacity-regulariser gradient once, one adam_step on the sum, and
    # accumulate_grad_stats once per view (densify.py:86-100)
    per_view = [_view_flat(orc, om, cams[v], targets[v], add_reg=(v == 0))
                for v in range(N_VIEWS)]
    full = sum(f for f, _ in per_view)
    err = float(np.abs(eng.reduced - full).max() / max(np.abs(full).max(), 1e-30))
    ref = om.copy()
    g, _ = _unflat(orc, full, len(ref))
    orc.adam(ref, g, orc.OAdam.for_map(ref))
    for _, gv in per_view:
        orc.accumulate_grad_stats(ref, gv)
    post = eng.gmap
    same_as_oracle = all(np.allclose(getattr(post, f), getattr(ref, f), rtol=0, atol=1e-12)
                         for f in ("positions", "rotations", "log_scales", "opacity_logits",
                                   "sh", "grad2d_accum", "grad3d_accum"))
    same_as_oracle &= bool(np.array_equal(post.obs_count, ref.obs_count))
    same = checksums_agree([post.positions, post.rotations, post.log_scales,
                            post.opacity_logits, post.sh, post.grad2d_accum, post.obs_count])
    out_q.put((rank, err, same, shard_views(N_VIEWS, rank, WORLD), same_as_oracle))
    dist.destroy_process_group()


def test_sharded_mapper_equals_batch_oracle_and_replicas_agree():
    """ShardedMapper over gloo (world 2) with the product's flat layout: the
    reduced buffer equals the single-process sum over all views, the update
    equals one oracle adam_step + accumulate_grad_stats on that sum, and the
    two replicas are byte-identical afterwards."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert [r[3] for r in res] == [[0, 2], [1]]
    for rank, err, same, _, ok in res:
        assert err < 1e-12, (rank, err)
        assert same, rank
        assert ok, rank


def test_flat_layout_matches_engine_planes():
    """The layout is plane-major with the 2-float flag tail; SH rest only
    above degree 0."""
    from paper_2410_00486_b200.distributed import FLAT_TAIL, flat_layout
    lay0, t0 = flat_layout(10, 0)
    lay3, t3 = flat_layout(10, 3)
    assert t0 == 10 * 20 + FLAT_TAIL and t3 == 10 * 65 + FLAT_TAIL
    offs = [off for _, _, off in lay3]
    assert offs == sorted(offs) and offs[0] == 0
    assert dict((nm, k) for nm, k, _ in lay0)["sh_rest"] == 0


@pytest.mark.parametrize("n_views,world", [(8, 1), (8, 2), (8, 4), (8, 8), (3, 4)])
def test_shard_views_partition(n_views, world):
    from paper_2410_00486_b200.distributed import shard_views
    shards = [shard_views(n_views, r, world) for r in range(world)]
    flat = sorted(v for s in shards for v in s)
    assert flat == list(range(n_views))
    assert 0 in shards[0]
