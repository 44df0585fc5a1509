"""BASELINE.json config 4 checked in full: every one of
the ~10,000 candidate-pair cones of the benchmark batch, run as ONE batched
device verdict, against the CPU oracle's single-worker run (es.py:252-339
restated; pinned to the reference by tests/test_oracle.py): verdict,
minimum-index witness and patterns_evaluated, bit for bit."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_06627_b200 import cones

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def batch():
    return cones.config4_batch(10_000)


@pytest.fixture(scope="module")
def oracle_results(batch):
    return O.run_packed_batch([batch.packed(i) for i in range(len(batch))])


def _compare(batch, rec, refs):
    verdicts = {"EXHAUSTED_ZERO": 0, "COUNTEREXAMPLE": 1}
    bad = []
    for i, g in enumerate(refs):
        got = (int(rec["verdict"][i]), int(rec["witness_index"][i]) if rec["verdict"][i] == 1 else None,
               int(rec["patterns_evaluated"][i]))
        want = (verdicts[g.verdict], g.witness_index, g.patterns_evaluated)
        if got != want:
            bad.append((i, got, want))
    return bad


@pytest.mark.parametrize("engine", ["auto", "interp"])
def test_config4_all_cones_match_oracle(gpu, batch, oracle_results, engine):
    assert len(batch) == 10_000
    rec = batch.run_arrays(engine=engine)
    bad = _compare(batch, rec, oracle_results)
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"
    assert np.all(rec["witness_minimal"][rec["verdict"] == 1] == 1)


def test_config4_repeatable(gpu, batch, oracle_results):
    """Three back-to-back batched verdicts (programs cached after the first)."""
    for _ in range(3):
        assert not _compare(batch, batch.run_arrays(), oracle_results)


def test_config4_eq_heavy_sweep_round(gpu):
    """The EQ-heavy variant: the sweep's own candidate pairs
    after a 64-word simulation of the configs[2] miter (sweep.py:313-345),
    mostly EQ cones swept to exhaustion, every result against the oracle."""
    b = cones.sweep_round_batch()
    refs = O.run_packed_batch([b.packed(i) for i in range(len(b))])
    rec = b.run_arrays()
    assert not _compare(b, rec, refs)
    assert int((rec["verdict"] == 0).sum()) > len(b) // 2  # EQ-heavy
