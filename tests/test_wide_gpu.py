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
