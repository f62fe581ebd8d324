"""Keyframe-sharded step on CPU: world_size 2 over gloo.

Each rank computes the oracle gradients of its shard of the views into the
engine's flat layout, the buffers are all-reduced, and every rank applies
the same Adam step.  Checks: the reduced buffer equals the single-process
sum over all views (the builder-defined batch oracle, A17), and the
replicas are byte-identical after the update.
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


def _flat(g, contributed_views):
    """Oracle grads of one view -> the engine's flat layout (SH degree 0):
    position 3N | rotation 4N | log_scale 3N | opacity N | sh_dc 3N |
    pos2d N | stat_g2d N | stat_g3d 3N | stat_cnt N."""
    seen = contributed_views.astype(np.float64)
    parts = [g.position.reshape(-1), g.rotation.reshape(-1), g.log_scale.reshape(-1),
             g.opacity_logit.reshape(-1), g.sh[:, 0, :].reshape(-1), g.pos2d_grad_norm,
             g.pos2d_grad_norm * seen, (g.position * seen[:, None]).reshape(-1), seen]
    return np.concatenate(parts)


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


def _worker(rank, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2410_00486_b200.distributed import (allreduce_sum, checksums_agree,
                                                   shard_views)
    orc, om, cams, targets = _scene()
    n = len(om)
    mine = shard_views(N_VIEWS, rank, WORLD)
    local = None
    for v in mine:
        f, _ = _view_flat(orc, om, cams[v], targets[v], add_reg=(v == 0))
        local = f if local is None else local + f
    buf = torch.from_numpy(local if local is not None else np.zeros(21 * n)).double()
    allreduce_sum(buf)
    reduced = buf.numpy()
    # single-process oracle of the batch: sum of all views, reg added once
    full = sum(_view_flat(orc, om, cams[v], targets[v], add_reg=(v == 0))[0]
               for v in range(N_VIEWS))
    err = float(np.abs(reduced - full).max() / max(np.abs(full).max(), 1e-30))
    # identical Adam step on every rank from the reduced gradients
    g = orc.OGrads(reduced[:3 * n].reshape(n, 3), reduced[3 * n:7 * n].reshape(n, 4),
                   reduced[7 * n:10 * n].reshape(n, 3), reduced[10 * n:11 * n],
                   np.concatenate([reduced[11 * n:14 * n].reshape(n, 1, 3),
                                   np.zeros((n, 15, 3))], axis=1),
                   reduced[14 * n:15 * n], reduced[20 * n:21 * n] > 0)
    st = orc.OAdam.for_map(om)
    orc.adam(om, g, st)
    same = checksums_agree([om.positions, om.rotations, om.log_scales, om.opacity_logits, om.sh])
    out_q.put((rank, err, same, mine))
    dist.destroy_process_group()


def test_sharded_allreduce_equals_batch_oracle_and_replicas_agree():
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
    for rank, err, same, _ in res:
        assert err < 1e-12, (rank, err)
        assert same, rank


@pytest.mark.parametrize("n_views,world", [(8, 1), (8, 2), (8, 4), (8, 8), (3, 4)])
def test_shard_views_partition(n_views, world):
    from paper_2410_00486_b200.distributed import shard_views
    shards = [shard_views(n_views, r, world) for r in range(world)]
    flat = sorted(v for s in shards for v in s)
    assert flat == list(range(n_views))
    assert 0 in shards[0]
