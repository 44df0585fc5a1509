"""GPU offload of ES inside the hybrid scheduler.

The reference reserves ``EnginePlan.es_on_device`` (sched.py:70, "never
set") and the paper states the rule: GPU ES is modelled
as 128 CPU threads and enabled when its predicted time exceeds 0.1 s; then
ES runs on the GPU, one CPU thread goes to BDD and the rest to SAT,
otherwise the CPU-only allocation applies (sched.py:175-207).  This module
implements that rule and the race (sched.py:210-266) with the ES racer on
the B200 engine; SAT and BDD stay the caller's (the reference's
``sat_check`` / ``bdd_check``, or any callable with the same contract).

    plan = plan_allocation(n, predictions, cutoff, gpu=True)
    result = dispatch(sm, plan, sat=ref.sat_check, bdd=ref.bdd_check)
"""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor, as_completed
from dataclasses import dataclass
from typing import Callable

from .verdict import UNKNOWN, CheckResult

# sched.py:23-28
ALPHA = 0.0003
BETA = 23
GAMMA = 1.5
PHI = 0.8
EASY_ES_PER_THREAD = 0.1
PRED_CAP = 1200.0
# PAPER.md:401-402
GPU_THREAD_EQUIV = 128
GPU_ENABLE_S = 0.1


@dataclass(frozen=True)
class Predictions:
    """sched.py:52-63 (capped at PRED_CAP)."""

    t_sat: float
    t_bdd: float
    t_es: float

    def __post_init__(self) -> None:
        for name in ("t_sat", "t_bdd", "t_es"):
            v = getattr(self, name)
            if not (v >= 0.0):
                raise ValueError(f"{name} must be >= 0, got {v}")
            object.__setattr__(self, name, min(float(v), PRED_CAP))


@dataclass(frozen=True)
class EnginePlan:
    """sched.py:66-71, with es_on_device actually used."""

    sat_threads: int = 0
    es_threads: int = 0
    bdd_threads: int = 0
    es_on_device: bool = False
    selected_single: str | None = None


def analytic_es_time(num_gates: int, num_pis: int, alpha: float = ALPHA, beta: int = BETA) -> float:
    """sched.py:35-39: single-thread CPU ES estimate."""
    return alpha * num_gates * 2.0 ** (num_pis - beta)


def device_es_time(num_gates: int, num_pis: int) -> float:
    """This engine's estimate on one B200 (seconds): the better of the
    interpreter (~1e14 gate-patterns/s with cofactor copies) and the K1
    kernel built directly as SASS (~2 ms from program to loaded module,
    then ~1.2e15 gate-patterns/s at k = 0 -- DESIGN §3 K1-direct)."""
    work = float(num_gates) * 2.0 ** num_pis
    return min(work / 1e14, 0.002 + work / 1.2e15)


def selection_plan(cost_sat: float, cost_es: float, n: int) -> EnginePlan:
    """sched.py:162-172: n == 1, pick by the XOR score."""
    if cost_sat <= cost_es:
        return EnginePlan(sat_threads=n, selected_single="SAT")
    return EnginePlan(es_threads=n, selected_single="ES")


def plan_allocation(n: int, p: Predictions, cutoff: float, cost_sat: float = 0.0,
                    cost_es: float = 1.0, gpu: bool = False) -> EnginePlan:
    """sched.py:175-207, plus the paper's GPU rule when ``gpu`` is True."""
    if n < 1:
        raise ValueError("need at least one thread")
    if p.t_es / n <= EASY_ES_PER_THREAD:
        return EnginePlan(es_threads=n, selected_single="ES" if n == 1 else None)
    if gpu and p.t_es / GPU_THREAD_EQUIV > GPU_ENABLE_S:
        # ES on the device; one CPU thread to BDD (when SAT keeps one), the rest SAT
        bdd = 1 if n >= 2 else 0
        return EnginePlan(sat_threads=n - bdd, bdd_threads=bdd, es_on_device=True)
    if n == 1:
        return selection_plan(cost_sat, cost_es, 1)
    es_ok = p.t_es / n <= GAMMA * cutoff
    bdd_ok = p.t_bdd < PHI * p.t_sat
    rho = p.t_sat / (n * p.t_es)
    if rho < 0.5:
        es = 1 if es_ok else 0
        bdd = 1 if bdd_ok and n - es >= 2 else 0
        return EnginePlan(sat_threads=n - es - bdd, es_threads=es, bdd_threads=bdd)
    if rho <= 2.0:
        es = n // 2 if es_ok else 0
        sat = n - es
        bdd = 0
        if bdd_ok and sat >= 2:
            sat -= 1
            bdd = 1
        return EnginePlan(sat_threads=sat, es_threads=es, bdd_threads=bdd)
    bdd = 1 if bdd_ok else 0
    if es_ok:
        return EnginePlan(sat_threads=1, bdd_threads=bdd, es_threads=n - 1 - bdd)
    return EnginePlan(sat_threads=n - bdd, bdd_threads=bdd)


def race(jobs: dict[str, Callable[[Callable[[], bool]], CheckResult]]) -> CheckResult:
    """Run every engine job at once; the first decisive verdict (EQUIVALENT /
    COUNTEREXAMPLE) wins and raises the shared cancel predicate the others
    poll (the B200 ES engine mirrors it into its native cancel flag, checked
    between launch slices).  The call returns once every engine has stopped,
    so no engine outlives its race.  Without a decisive verdict the result is
    UNKNOWN, reason "timeout" if any engine timed out, with each engine's
    statistics -- the reference race's outcome contract (sched.py:210-266).
    A job that raises counts as UNKNOWN("error: ...")."""
    stop = threading.Event()
    first = threading.Lock()
    winner: list[CheckResult] = []

    def guarded(name, job):
        try:
            r = job(stop.is_set)
        except Exception as exc:  # an engine bug must not hang the race
            r = CheckResult(UNKNOWN, reason=f"error: {exc}", engine=name)
        if r.verdict != UNKNOWN:
            with first:  # the first decisive verdict to land wins ...
                if not winner:
                    winner.append(r)
            stop.set()  # ... and cancels the others right away
        return r

    undecided: dict[str, CheckResult] = {}
    with ThreadPoolExecutor(max_workers=len(jobs), thread_name_prefix="race") as pool:
        futs = {pool.submit(guarded, name, job): name for name, job in jobs.items()}
        for fut in as_completed(futs):  # every engine has stopped when the pool closes
            r = fut.result()
            if r.verdict == UNKNOWN:
                undecided[r.engine or futs[fut]] = r
    if winner:
        return winner[0]
    reasons = {r.reason for r in undecided.values()}
    reason = "timeout" if "timeout" in reasons else (min(reasons) if reasons else "")
    return CheckResult(UNKNOWN, reason=reason,
                       stats={"engines": {k: dict(r.stats, reason=r.reason) for k, r in undecided.items()}})


def dispatch(sm, plan: EnginePlan, sat: Callable | None = None, bdd: Callable | None = None,
             es_cpu: Callable | None = None, budget: float | None = None, seed: int = 0,
             device: int = 0) -> CheckResult:
    """The planned engines raced on ``sm`` (the reference's dispatch contract,
    sched.py:210-266).  ES runs on the B200 (es.es_check) when the plan says
    es_on_device -- or whenever no CPU ES callable is given; SAT and BDD are
    the caller's callables with the reference's signatures
    (sat(sm, threads=, budget=, cancel=, seed=), bdd(sm, budget=, cancel=),
    es_cpu(sm, workers=, budget=, cancel=))."""
    from . import es as gpu_es

    jobs: dict[str, Callable[[Callable[[], bool]], CheckResult]] = {}
    if plan.sat_threads > 0:
        if sat is None:
            raise ValueError("plan enables SAT but no sat callable was given")
        jobs["sat"] = lambda cancel: sat(sm, threads=plan.sat_threads, budget=budget, cancel=cancel,
                                         seed=seed)
    if plan.es_on_device or (plan.es_threads > 0 and es_cpu is None):
        jobs["es"] = lambda cancel: gpu_es.es_check(sm, budget=budget, cancel=cancel, device=device)
    elif plan.es_threads > 0:
        jobs["es"] = lambda cancel: es_cpu(sm, workers=plan.es_threads, budget=budget, cancel=cancel)
    if plan.bdd_threads > 0:
        if bdd is None:
            raise ValueError("plan enables BDD but no bdd callable was given")
        jobs["bdd"] = lambda cancel: bdd(sm, budget=budget, cancel=cancel)
    if not jobs:
        raise ValueError("plan enables no engine")
    return race(jobs)
