"""Programs whose live set does not fit the K2 interpreter's shared memory
are routed to K1 by engine='auto' (single runs and batches) instead of
failing; engine='interp' says so explicitly."""
import pytest

from oracle import oracle as O
from paper_2512_06627_b200 import _native as N
from paper_2512_06627_b200 import es
from tests.wide_circuits import butterfly

SMEM_LIMIT = 232448  # B200 opt-in shared memory per CTA


@pytest.fixture(scope="module")
def wide():
    return {eq: butterfly(eq=eq) for eq in (False, True)}


def test_wide_live_set_exceeds_k2(wide):
    for x in wide.values():
        p = es.compile_program(x)
        assert es.k2_stats(p)["slots"] * 512 > SMEM_LIMIT


@pytest.mark.gpu
@pytest.mark.parametrize("eq", [False, True])
def test_auto_routes_wide_program_to_k1(gpu, wide, eq):
    x = wide[eq]
    ref = O.run_exhaustive(O.compile_program(x), workers=1)
    r = es.run_exhaustive(es.compile_program(x), engine="auto")
    assert r.stats["engine"] == "jit"
    assert (r.verdict, r.witness_index, r.patterns_evaluated) == \
        (ref.verdict, ref.witness_index, ref.patterns_evaluated)
    c = es.es_check(type("S", (), {"circuit": x})())
    assert c.verdict == ("EQUIVALENT" if eq else "COUNTEREXAMPLE")


@pytest.mark.gpu
def test_batch_routes_wide_program_to_k1(gpu, wide):
    from paper_2512_06627_b200 import miter as M
    small = M.gen_adder_miter(6)
    progs = [es.compile_program(x) for x in (small, wide[False], wide[True])]
    refs = [O.run_exhaustive(O.compile_program(x), workers=1) for x in (small, wide[False], wide[True])]
    res = es.run_exhaustive_batch(progs)
    for r, g in zip(res, refs):
        assert (r.verdict, r.witness_index, r.patterns_evaluated) == \
            (g.verdict, g.witness_index, g.patterns_evaluated)
    assert res[1].stats["engine"] == "jit" and res[0].stats["engine"] == "interp"


@pytest.mark.gpu
def test_forced_interp_rejects_wide_program(gpu, wide):
    with pytest.raises(N.NativeError, match="too many for the K2 interpreter"):
        es.run_exhaustive(es.compile_program(wide[True]), engine="interp")
