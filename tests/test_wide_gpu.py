"""Beyond the reference's reach (its CPU ES needs hours at 36 PIs): size-
independent properties at 36 PIs on the GPU.  An EQ miter must exhaust 2^36
patterns; a miter with a single failing pattern (a minterm ORed into the
output) must return exactly that pattern as the minimum-index witness, for
every K1 cofactor mode."""
import pytest

from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M
from tests.golden import recipes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mult18():
    return M.gen_multiplier_miter(18, "array", "booth")


@pytest.mark.parametrize("cof", ["auto", "throughput", 2])
def test_36_pi_equivalent(gpu, mult18, cof):
    r = es.run_exhaustive(es.compile_program(mult18), engine="jit", cofactor=cof)
    assert r.verdict == es.EXHAUSTED_ZERO and r.patterns_evaluated == 1 << 36


@pytest.mark.parametrize("needle", [0xABCDE1234, (1 << 36) - 1, 1 << 35, 7])
def test_36_pi_single_failing_pattern(gpu, needle):
    x = recipes.build_sweep_circuit({"kind": "mult", "width": 18, "a": "array", "b": "booth",
                                     "needle": needle})
    p = es.compile_program(x)
    for cof in ("none", "throughput"):
        r = es.run_exhaustive(p, engine="jit", cofactor=cof)
        assert r.verdict == es.ES_COUNTEREXAMPLE and r.witness_index == needle, (cof, r.witness_index)
        b = min(36, 14)
        assert r.patterns_evaluated == ((needle >> b) + 1) << b
    assert M.evaluate(x, r.witness) == 1


def test_stopped_cofactored_sweep_flags_unproven_minimum(gpu):
    """A cancel that stops a cofactored sweep after a witness above the swept
    prefix keeps the (valid) witness but does not claim it is the minimum
    (ADVICE r01, medium): witness_minimal is False and patterns_evaluated is
    what was swept.  A run that finishes first must return the needle."""
    import time

    needle = 1 << 35
    x = recipes.build_sweep_circuit({"kind": "mult", "width": 18, "a": "array", "b": "booth",
                                     "needle": needle})
    p = es.compile_program(x)
    es.run_exhaustive(p, engine="jit", cofactor=4, budget=0.001)  # JIT outside the timed call
    t0 = time.monotonic()
    r = es.run_exhaustive(p, engine="jit", cofactor=4, slice_ms=0.5,
                          cancel=lambda: time.monotonic() - t0 > 0.004)
    if r.verdict == es.BUDGET_EXCEEDED:
        assert r.patterns_evaluated < 1 << 36
        return
    assert r.verdict == es.ES_COUNTEREXAMPLE and M.evaluate(x, r.witness) == 1
    if r.stats["witness_minimal"]:
        assert r.witness_index == needle
    else:
        assert r.patterns_evaluated == r.stats["patterns_swept"] < 1 << 36
