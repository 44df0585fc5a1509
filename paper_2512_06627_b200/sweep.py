"""SAT-sweeping with the exact-simulation engine on the GPU.

The reference's sweep (cecprove/sweep.py:292-409) with ``engine="es"``
checks candidate pairs one at a time: extract the cone-local sub-miter
(sweep.py:92-158), ``es_check`` it (sweep.py:240-243), merge or refine, and
finally discharge the output obligation.  Here every step runs on the B200
path and the pairs are checked in rounds:

  random simulation + PE classes   K3 (sim.pe_classes; sweep.py:313-345)
  first-round refutation           the same simulated words (sweep.py:318-330)
  pair extraction                  C++, multithreaded (es_batch_extract)
  pair checks                      ONE batched K2 launch per round (es_batch_run)
  refinement                       K3 (sim.refine_with_cex; sweep.py:161-193)
  final obligation                 es_check (K1 or K2; sweep.py:382-405)

A round extracts every open pair of the current classes against the merges
known at its start (the reference extracts each pair against the merges of
all earlier pairs), so intermediate sub-miters may be larger; merges are
proven equivalences either way, so the final obligation -- and the verdict --
is the reference's.  Counterexamples of a round refine the classes in
discovery order before the next round.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import es, sim
from .cones import NativeBatch
from .miter import evaluate
from .verdict import COUNTEREXAMPLE, EQUIVALENT, UNKNOWN, CheckResult
from .xag import Lit

_ONES = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass
class SweepConfig:
    """The ES-relevant fields of sweep.py:197-208."""

    engine: str = "es"
    budget: float | None = None  # global wall budget
    pair_budget: float = 5.0  # per sub-miter (a round of n gets n x); final obligation gets the rest
    seed: int = 0
    sim_words: int = 64
    device: int = 0


def _expand(pi_map, witness_index: int, num_pis: int) -> tuple[int, ...]:
    bits = [0] * num_pis
    for i, orig in enumerate(pi_map):
        bits[orig - 1] = (witness_index >> i) & 1
    return tuple(bits)


def sweep(miter, config: SweepConfig = SweepConfig()) -> CheckResult:
    """Full sweeping run on a single-output miter, ES on the GPU."""
    if config.engine != "es":
        raise ValueError("the B200 sweep drives the exact-simulation engine only (engine='es')")
    t0 = time.monotonic()
    deadline = None if config.budget is None else t0 + config.budget
    stats = {"engine_calls": 0, "merges": 0, "structural_merges": 0, "refinements": 0,
             "unknown_pairs": 0, "sim_patterns": 0, "rounds": 0}

    def finish(res: CheckResult) -> CheckResult:
        stats["wall_time"] = time.monotonic() - t0
        res.stats = {**res.stats, **stats}
        return res

    def remaining() -> float | None:
        return None if deadline is None else deadline - time.monotonic()

    merges: dict[int, Lit] = {}
    attempted: set[tuple[int, int]] = set()
    dev = config.device

    pi_words = sim.random_pi_words(miter.num_pis, config.sim_words, config.seed)
    vals = sim.simulate(miter, pi_words, dev)
    stats["sim_patterns"] = config.sim_words * 64
    out = miter.output
    out_word = vals[out.node] ^ (_ONES if out.neg else np.uint64(0))
    hit = np.flatnonzero(out_word)
    if hit.size:  # the first simulation round doubles as a refutation attempt
        w = int(hit[0])
        b = int(out_word[w]).bit_length() - 1
        pattern = tuple(int(pi_words[i, w] >> np.uint64(b)) & 1 for i in range(miter.num_pis))
        if evaluate(miter, pattern) != 1:
            raise AssertionError("simulation witness failed re-check")
        return finish(CheckResult(COUNTEREXAMPLE, witness=pattern, engine="sim"))
    classes = sim.pe_classes(miter, pi_words=pi_words, device=dev)

    while True:
        pairs = []
        for cls in classes:
            rep = cls.representative
            rep_pol = next(p for n, p in cls.members if n == rep)
            for node, pol in cls.members:
                if node == rep or node in merges or (rep, node) in attempted:
                    continue
                pairs.append((rep, node, pol != rep_pol))
        if not pairs:
            break
        rem = remaining()
        if rem is not None and rem <= 0:
            return finish(CheckResult(UNKNOWN, reason="timeout"))
        stats["rounds"] += 1
        batch = NativeBatch(miter, pairs, merges)
        tab = batch.table()
        # constant sub-miters are settled structurally (sweep.py:347-353)
        run_idx = []
        for i, (rep, node, rel) in enumerate(pairs):
            if tab["num_gates"][i] == 0:
                sm = batch.submiter(i)
                o = sm.circuit.output
                if o.node == 0:
                    if o.neg:
                        attempted.add((rep, node))
                    else:
                        merges[node] = Lit(rep, rel)
                        stats["structural_merges"] += 1
                    continue
            run_idx.append(i)
        if not run_idx:
            continue
        batch.select(run_idx)
        # the reference gives each sub-miter pair_budget (sweep.py:355-356)
        budget = config.pair_budget * len(run_idx)
        budget = budget if rem is None else min(budget, rem)
        # the interpreter's cofactor-depth search costs more host time than it
        # saves on a round's few dozen cones: plain programs, unless the round
        # is heavy (its big jobs go through K1 either way)
        work = float((tab["G"].astype(np.float64)[run_idx] * np.exp2(tab["num_pis"][run_idx])).sum())
        results = batch.run(budget=budget, device=dev, cofactor="auto" if work > 1e13 else "none")
        stats["engine_calls"] += len(run_idx)
        cexes = []
        for j, (k, r) in enumerate(zip(run_idx, results)):
            rep, node, rel = pairs[k]
            if r is not None and r.verdict == es.EXHAUSTED_ZERO:
                if node not in merges:
                    merges[node] = Lit(rep, rel)
                    stats["merges"] += 1
            elif r is not None and r.verdict == es.ES_COUNTEREXAMPLE:
                pi_map = batch.submiter(j).pi_map
                cexes.append(_expand(pi_map, r.witness_index, miter.num_pis))
                attempted.add((rep, node))
            else:
                attempted.add((rep, node))
                stats["unknown_pairs"] += 1
        for pattern in cexes:
            classes = sim.refine_with_cex(miter, classes, pattern, dev)
            stats["refinements"] += 1
        batch.close()

    # final obligation: the output against constant zero (sweep.py:382-405)
    final_batch = NativeBatch(miter, [(out.node, 0, bool(out.neg))], merges)
    final = final_batch.submiter(0)
    o = final.circuit.output
    if o.node == 0:
        if not o.neg:
            return finish(CheckResult(EQUIVALENT, engine="sweep"))
        pattern = (0,) * miter.num_pis
        if evaluate(miter, pattern) != 1:
            raise AssertionError("constant-one discharge failed re-check")
        return finish(CheckResult(COUNTEREXAMPLE, witness=pattern, engine="sweep"))
    res = es.es_check(final, budget=remaining(), device=dev)
    stats["engine_calls"] += 1
    if res.verdict == EQUIVALENT:
        return finish(CheckResult(EQUIVALENT, engine=res.engine, stats=res.stats))
    if res.verdict == COUNTEREXAMPLE:
        idx = sum(b << i for i, b in enumerate(res.witness))
        pattern = _expand(final.pi_map, idx, miter.num_pis)
        if evaluate(miter, pattern) != 1:
            raise AssertionError("sweep witness failed re-check")
        return finish(CheckResult(COUNTEREXAMPLE, witness=pattern, engine=res.engine, stats=res.stats))
    return finish(CheckResult(UNKNOWN, reason=res.reason or "timeout", engine=res.engine,
                              stats=res.stats))
