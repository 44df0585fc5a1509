"""GPU offload inside the hybrid scheduler (offload.py; sched.py:175-266,
PAPER.md:401-402).  The CPU-only rules are checked against the reference's
plan_allocation on a grid of predictions (imported when the reference is
present: the build container); the GPU rule and the race are checked with
stand-in SAT/BDD engines."""
import itertools
import time

import pytest

from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200 import offload as O
from paper_2512_06627_b200.verdict import COUNTEREXAMPLE, EQUIVALENT, UNKNOWN, CheckResult

GRID = list(itertools.product([1, 2, 3, 8, 32], [0.01, 0.5, 10.0, 900.0], [0.02, 1.0, 50.0],
                              [0.001, 0.3, 7.0, 2000.0], [5.0, 60.0]))


def test_cpu_rules_match_reference():
    import os
    import sys
    src = "/root/reference/pkg/src"  # the build container only (never on the GPU box)
    if os.path.isdir(src) and src not in sys.path:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
        sys.path.append(src)
    ref = pytest.importorskip("cecprove.sched", reason="reference not importable here")
    for n, ts, tb, te, cutoff in GRID:
        p = O.Predictions(ts, tb, te)
        rp = ref.Predictions(ts, tb, te)
        for cs, ce in ((0.0, 1.0), (3.0, 1.0)):
            a = O.plan_allocation(n, p, cutoff, cs, ce, gpu=False)
            b = ref.plan_allocation(n, rp, cutoff, cs, ce)
            assert (a.sat_threads, a.es_threads, a.bdd_threads, a.selected_single) == \
                (b.sat_threads, b.es_threads, b.bdd_threads, b.selected_single), (n, ts, tb, te)
            assert not a.es_on_device


def test_gpu_rule():
    # t_es / 128 > 0.1 s -> ES on the device, one BDD thread, the rest SAT
    p = O.Predictions(100.0, 100.0, 13.0)
    plan = O.plan_allocation(8, p, 60.0, gpu=True)
    assert plan.es_on_device and plan.bdd_threads == 1 and plan.sat_threads == 7 and plan.es_threads == 0
    # below the bar: the CPU-only allocation
    p = O.Predictions(100.0, 100.0, 12.0)
    assert O.plan_allocation(8, p, 60.0, gpu=True) == O.plan_allocation(8, p, 60.0, gpu=False)
    # easy instances stay ES-only on the CPU plan (sched.py:180-182)
    p = O.Predictions(100.0, 100.0, 0.5)
    assert O.plan_allocation(8, p, 60.0, gpu=True).es_threads == 8
    assert O.plan_allocation(1, O.Predictions(1, 1, 20.0), 60.0, gpu=True).sat_threads == 1


def test_device_estimate_orders():
    assert O.device_es_time(2833, 32) < O.analytic_es_time(2833, 32) / 100
    assert O.device_es_time(100, 14) < 0.001


def _slow_sat(sm, threads, budget, cancel, seed):
    t = time.monotonic()
    while not cancel() and time.monotonic() - t < 20:
        time.sleep(0.001)
    return CheckResult(UNKNOWN, reason="cancelled", engine="sat")


def _fast_sat(verdict):
    def sat(sm, threads, budget, cancel, seed):
        return CheckResult(verdict, engine="sat")
    return sat


def _bdd(sm, budget, cancel):
    return CheckResult(UNKNOWN, reason="memout", engine="bdd")


class _SM:
    def __init__(self, x):
        self.circuit = x


@pytest.mark.gpu
def test_race_gpu_es_wins(gpu):
    m = M.gen_multiplier_miter(10, "array", "booth")
    plan = O.EnginePlan(sat_threads=7, bdd_threads=1, es_on_device=True)
    t = time.monotonic()
    r = O.dispatch(_SM(m), plan, sat=_slow_sat, bdd=_bdd)
    assert r.verdict == EQUIVALENT and r.engine == "es"
    assert time.monotonic() - t < 10  # the GPU verdict cancelled the SAT racer
    bad = M.flip_gate(m, 200)
    r = O.dispatch(_SM(bad), plan, sat=_slow_sat, bdd=_bdd)
    assert r.verdict == COUNTEREXAMPLE and M.evaluate(bad, r.witness) == 1


@pytest.mark.gpu
def test_race_sat_wins_and_cancels_gpu(gpu):
    m = M.gen_multiplier_miter(16, "array", "booth")
    plan = O.EnginePlan(sat_threads=1, es_on_device=True)
    r = O.dispatch(_SM(m), plan, sat=_fast_sat(EQUIVALENT))
    assert r.verdict == EQUIVALENT
