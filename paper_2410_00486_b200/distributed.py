"""Keyframe-sharded multi-GPU mapping (builder-defined batch
semantics A17 -- the reference trains one view per step, trainer.py:194-207).

One process per GPU.  A step takes a batch of V keyframe views of the
replicated map: rank r renders and back-propagates views r, r+W, ... into
one flat per-Gaussian buffer (parameter gradients + densify-statistics
increments, see MappingEngine._flat_grads), the buffers are summed with a
single all-reduce (NCCL over NVLink on B200, gloo in the CPU tests), and
every rank applies the identical Adam step.  All ranks receive the same
reduced bytes, so the replicas stay bit-identical; ``replica_checksum``
verifies that.
"""

from __future__ import annotations

import hashlib

import numpy as np
import torch
import torch.distributed as dist


# The flat per-Gaussian buffer one keyframe-batch step sums over views and
# ranks: plane name -> floats per Gaussian, planes stored one
# after another (plane-major, each N x k), then FLAT_TAIL floats written by
# ss_status_flags (any pair overflow, any error) so the gradient all-reduce
# also tells every rank whether some rank has to redo the step or raise.
FLAT_PLANES = (("position", 3), ("rotation", 4), ("log_scale", 3), ("opacity", 1),
               ("sh_dc", 3), ("sh_rest", 45), ("pos2d", 1), ("stat_g2d", 1), ("stat_g3d", 3),
               ("stat_cnt", 1))
FLAT_TAIL = 2


def flat_layout(n: int, sh_degree: int):
    """[(plane, floats per Gaussian, offset in floats)] of the flat buffer
    for a map of n Gaussians, and its total length in floats (tail
    included).  sh_rest is absent (0 floats) at SH degree 0."""
    out, off = [], 0
    for name, k in FLAT_PLANES:
        if name == "sh_rest" and sh_degree == 0:
            k = 0
        out.append((name, k, off))
        off += k * n
    return out, off + FLAT_TAIL


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Round-robin view assignment: rank r gets r, r + world, ..."""
    return list(range(rank, n_views, world))


def allreduce_sum(buf: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over ranks (one collective per step)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def replica_checksum(arrays) -> str:
    """SHA-1 over the raw bytes of a map's arrays (replica identity check)."""
    h = hashlib.sha1()
    for a in arrays:
        if isinstance(a, torch.Tensor):
            a = a.detach().contiguous().cpu().numpy()
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def checksums_agree(arrays, group=None) -> bool:
    """True when every rank holds byte-identical arrays."""
    mine = replica_checksum(arrays)
    if not (dist.is_available() and dist.is_initialized()):
        return True
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, mine, group=group)
    return all(x == mine for x in out)


class ShardedMapper:
    """Drives a MappingEngine through keyframe-batch steps on one rank."""

    def __init__(self, engine, rank: int | None = None, world: int | None = None, group=None):
        self.engine = engine
        ok = dist.is_available() and dist.is_initialized()
        self.rank = rank if rank is not None else (dist.get_rank() if ok else 0)
        self.world = world if world is not None else (dist.get_world_size() if ok else 1)
        self.group = group

    def step(self, cameras, targets, target_depths=None):
        """One keyframe-batch step over all V views (each rank renders its shard)."""
        mine = shard_views(len(cameras), self.rank, self.world)
        cams = [cameras[i] for i in mine]
        tgts = [targets[i] for i in mine]
        tds = [target_depths[i] for i in mine] if target_depths is not None else None
        return self.engine.multiview_step(
            cams, tgts, tds, allreduce=lambda b: allreduce_sum(b, self.group),
            add_reg=(self.rank == 0))
