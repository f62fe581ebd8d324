"""Loss-adaptive keyframe scheduling around the mapping engine.

`KeyframeScheduler` restates scheduler.py:22-89: per keyframe a remaining
iteration budget and the last recorded loss; `select` draws uniformly among
keyframes with budget left and, once every budget is spent, refills 2
iterations for the max(1, k // d) largest losses (ties to the most recent
keyframe) and 1 for the rest; new keyframes enter with r0 and an infinite
loss.  Same numpy Generator stream, so the same seed selects the same ids
as the reference (tests/golden/scheduler_metrics.json).

`ScheduledMapper` drives a `MappingEngine` the way `_Trainer.train_one`
drives the reference (trainer.py:194-210).  The engine publishes a step's
loss two steps late without stalling the GPU (ss_step_snapshot), so the
budget is spent when a keyframe is selected and its loss is stored when it
arrives; `synchronous=True` waits for each loss instead and reproduces the
reference's select/record order exactly.
"""

from __future__ import annotations

import math

import numpy as np

LOSS_SENTINEL = math.inf


class KeyframeScheduler:
    """scheduler.py:22-89 (single-writer state machine owned by the trainer)."""

    def __init__(self, d: int = 4, r0: int = 8, seed: int = 0):
        if d < 1:
            raise ValueError("d must be >= 1")
        if r0 < 1:
            raise ValueError("r0 must be >= 1")
        self.d, self.r0 = int(d), int(r0)
        self.ids: list[int] = []
        self.remaining: list[int] = []
        self.last_loss: list[float] = []
        self.rng = np.random.default_rng(seed)
        self._pos: dict[int, int] = {}

    def __len__(self) -> int:
        return len(self.ids)

    def add_keyframe(self, keyframe_id: int) -> None:
        if keyframe_id in self._pos:
            raise ValueError(f"keyframe {keyframe_id} already present")
        self._pos[keyframe_id] = len(self.ids)
        self.ids.append(keyframe_id)
        self.remaining.append(self.r0)
        self.last_loss.append(LOSS_SENTINEL)

    def select(self) -> int:
        if not self.ids:
            raise ValueError("cannot select from an empty keyframe pool")
        live = [k for k, r in enumerate(self.remaining) if r > 0]
        if not live:
            self.refill()
            live = list(range(len(self.ids)))
        return self.ids[live[int(self.rng.integers(len(live)))]]

    def select_uniform_baseline(self) -> int:
        if not self.ids:
            raise ValueError("cannot select from an empty keyframe pool")
        return self.ids[int(self.rng.integers(len(self.ids)))]

    def spend(self, keyframe_id: int) -> None:
        """Take one iteration from the keyframe's budget."""
        k = self._pos[keyframe_id]
        if self.remaining[k] <= 0:
            raise ValueError(f"keyframe {keyframe_id} has no remaining iterations; "
                             "select() should have been used to pick it")
        self.remaining[k] -= 1

    def set_loss(self, keyframe_id: int, loss: float) -> None:
        self.last_loss[self._pos[keyframe_id]] = float(loss)

    def record_result(self, keyframe_id: int, loss: float) -> None:
        """Spend one iteration and store its loss (scheduler.py:62-71)."""
        self.spend(keyframe_id)
        self.set_loss(keyframe_id, loss)

    def refill(self) -> None:
        n = len(self.ids)
        if n == 0:
            return
        if any(r != 0 for r in self.remaining):
            raise ValueError("refill requires every remaining budget to be 0")
        top = max(1, n // self.d)
        rank = sorted(range(n), key=lambda k: (self.last_loss[k], k), reverse=True)
        boosted = set(rank[:top])
        self.remaining = [2 if k in boosted else 1 for k in range(n)]


class ScheduledMapper:
    """Keyframe-scheduled mapping iterations on a MappingEngine."""

    def __init__(self, engine, scheduler: KeyframeScheduler | None = None,
                 mode: str = "adaptive", synchronous: bool = False):
        if mode not in ("adaptive", "uniform"):
            raise ValueError("mode must be 'adaptive' or 'uniform'")
        self.engine = engine
        self.sched = scheduler if scheduler is not None else KeyframeScheduler()
        self.mode = mode
        self.synchronous = synchronous
        self.frames: dict[int, tuple] = {}
        self.kf_iters: dict[int, int] = {}
        self.kf_loss: dict[int, float] = {}
        self._pending: dict[int, int] = {}  # engine iteration -> keyframe id
        self._seen = 0                      # consumed entries of the engine's loss log

    def add_keyframe(self, keyframe_id: int, camera, target, target_depth=None) -> None:
        self.sched.add_keyframe(keyframe_id)
        self.frames[keyframe_id] = (camera, target, target_depth)
        self.kf_iters[keyframe_id] = 0

    def step(self) -> int:
        """One iteration on the selected keyframe; returns its id."""
        kf = self.sched.select() if self.mode == "adaptive" else \
            self.sched.select_uniform_baseline()
        if self.mode == "adaptive":
            self.sched.spend(kf)
        cam, tgt, tdep = self.frames[kf]
        index = self.engine.step(cam, tgt, tdep)
        self._pending[index] = kf
        self.kf_iters[kf] += 1
        if self.synchronous:
            self.engine.synchronize()
        self._consume()
        return kf

    def _consume(self) -> None:
        log = self.engine._loss_log
        while self._seen < len(log):
            index, total, _rendered = log[self._seen]
            self._seen += 1
            kf = self._pending.pop(index, None)
            if kf is None:
                continue
            self.kf_loss[kf] = total
            if self.mode == "adaptive":
                self.sched.set_loss(kf, total)

    def synchronize(self) -> None:
        self.engine.synchronize()
        self._consume()
