"""KeyframeScheduler (scheduler.py:22-89) against traces produced by the
reference itself (tests/golden/make_golden.py: capture_scheduler_and_metrics),
and the ScheduledMapper loss feed with a stub engine (CPU)."""

import json
import math
import os

import pytest

from paper_2410_00486_b200.scheduler import KeyframeScheduler, ScheduledMapper

GOLD = os.path.join(os.path.dirname(__file__), "golden", "scheduler_metrics.json")


def _loss_of(kf, step):
    return 1.0 / (1.0 + kf) + 0.01 * ((step * 7919) % 13)


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


@pytest.mark.parametrize("d,r0,seed", [(4, 8, 0), (2, 3, 7)])
def test_adaptive_selection_matches_reference(gold, d, r0, seed):
    sch = KeyframeScheduler(d=d, r0=r0, seed=seed)
    picks = []
    for step in range(240):
        if step % 10 == 0:
            sch.add_keyframe(step // 10)
        kf = sch.select()
        picks.append(kf)
        sch.record_result(kf, _loss_of(kf, step))
    assert picks == gold[f"select_d{d}_r{r0}_s{seed}"]
    assert sch.remaining == gold[f"remaining_d{d}_r{r0}_s{seed}"]


@pytest.mark.parametrize("d,r0,seed", [(4, 8, 0), (2, 3, 7)])
def test_uniform_baseline_matches_reference(gold, d, r0, seed):
    sch = KeyframeScheduler(d=d, r0=r0, seed=seed)
    for k in range(5):
        sch.add_keyframe(k)
    assert [sch.select_uniform_baseline() for _ in range(50)] == \
        gold[f"uniform_d{d}_r{r0}_s{seed}"]


def test_errors_and_refill_rule():
    with pytest.raises(ValueError):
        KeyframeScheduler(d=0)
    with pytest.raises(ValueError):
        KeyframeScheduler(r0=0)
    sch = KeyframeScheduler(d=2, r0=1, seed=0)
    with pytest.raises(ValueError):
        sch.select()
    for k in range(4):
        sch.add_keyframe(k)
    with pytest.raises(ValueError):
        sch.add_keyframe(2)
    with pytest.raises(ValueError):
        sch.refill()  # budgets not exhausted
    for k, loss in zip(range(4), [0.5, 0.9, 0.9, 0.1]):
        sch.record_result(k, loss)
    with pytest.raises(ValueError):
        sch.record_result(0, 0.1)  # no budget left
    sch.refill()
    # d_k = 2: the two largest losses, the tie resolved towards the newer keyframe
    assert sch.remaining == [1, 2, 2, 1]
    fresh = KeyframeScheduler()
    fresh.add_keyframe(9)
    assert math.isinf(fresh.last_loss[0]) and fresh.remaining == [8]


class _StubEngine:
    """Publishes a step's loss two steps late, like MappingEngine."""

    def __init__(self):
        self.iteration = 0
        self._loss_log = []
        self._queue = []

    def step(self, cam, target, target_depth=None):
        i = self.iteration
        self.iteration += 1
        self._queue.append((i, float(target), float(target)))
        while len(self._queue) > 2:
            self._loss_log.append(self._queue.pop(0))
        return i

    def synchronize(self):
        self._loss_log.extend(self._queue)
        self._queue.clear()


def test_scheduled_mapper_lagged_and_synchronous():
    # synchronous mode reproduces select/record_result order exactly
    ref = KeyframeScheduler(d=2, r0=2, seed=3)
    eng = _StubEngine()
    sm = ScheduledMapper(eng, KeyframeScheduler(d=2, r0=2, seed=3), synchronous=True)
    for k in range(3):
        ref.add_keyframe(k)
        sm.add_keyframe(k, None, 0.1 * (k + 1))
    for _ in range(30):
        a = ref.select()
        ref.record_result(a, 0.1 * (a + 1))
        assert sm.step() == a
    assert sm.sched.remaining == ref.remaining
    # lagged mode: budgets spent at selection, losses arrive two steps late
    eng = _StubEngine()
    sm = ScheduledMapper(eng, KeyframeScheduler(d=2, r0=2, seed=3))
    for k in range(3):
        sm.add_keyframe(k, None, 0.1 * (k + 1))
    for _ in range(5):
        sm.step()
    assert len(sm._pending) == 2
    sm.synchronize()
    assert not sm._pending
    assert sum(sm.kf_iters.values()) == 5
    assert all(sm.kf_loss[k] == pytest.approx(0.1 * (k + 1)) for k in sm.kf_loss)
