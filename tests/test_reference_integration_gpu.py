"""INTEGRATION.md Option A executed: the UNMODIFIED reference package
(cecprove, installed in baseline/_ref) with its ES entry points swapped for
the B200 engine, driven through the reference's OWN callers:

* cecprove.sweep.sweep(miter, SweepConfig(engine="es")) -> _check_submiter ->
  es_check (sweep.py:240-243) on the sweep fixtures the reference produced
  with its CPU ES (tests/golden/sweep_golden.json): same verdict, witness and
  sweep trajectory (engine calls, merges, refinements);
* cecprove.sched.dispatch with an ES-only and an ES+SAT plan
  (sched.py:210-266, es_check at :236-238);
* cecprove.es.run_exhaustive on the reference's own InstrProgram objects.
"""
import json
import os
import sys

import pytest

from paper_2512_06627_b200 import es as b200_es
from tests.golden import recipes

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
GOLD = os.path.join(ROOT, "tests", "golden", "sweep_golden.json")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "cecprove")):
        pytest.fail("baseline/_ref is missing: install the reference (DESIGN.md, reference arm)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import cecprove.es
    import cecprove.eval
    import cecprove.sched
    import cecprove.sweep
    import cecprove.xag

    orig = (cecprove.es.es_check, cecprove.es.run_exhaustive)
    # Option A: the reference looks es_check up at call time (sweep.py:241, sched.py:214)
    cecprove.es.es_check = b200_es.es_check
    cecprove.es.run_exhaustive = b200_es.run_exhaustive
    yield cecprove
    cecprove.es.es_check, cecprove.es.run_exhaustive = orig


def to_ref(x, ref):
    X = ref.xag
    return X.Xag(x.num_pis,
                 tuple(X.Gate(X.GateKind(int(g.kind)), X.Lit(g.in0.node, bool(g.in0.neg)),
                              X.Lit(g.in1.node, bool(g.in1.neg))) for g in x.gates),
                 tuple(X.Lit(o.node, bool(o.neg)) for o in x.outputs))


def test_reference_sweep_on_b200_engine(gpu, ref):
    rows = json.load(open(GOLD))["rows"]
    for row in rows:
        x = to_ref(recipes.build_sweep_circuit(row), ref)
        r = ref.sweep.sweep(x, ref.sweep.SweepConfig(engine="es"))
        assert (r.verdict, r.engine) == (row["verdict"], row["engine"]), row
        if row["witness"] is not None:
            assert list(r.witness) == row["witness"], row
        for k, v in row["stats"].items():
            assert r.stats[k] == v, (row, k)


def test_reference_dispatch_on_b200_engine(gpu, ref):
    from paper_2512_06627_b200 import miter as M
    good = to_ref(M.gen_multiplier_miter(10, "array", "wallace"), ref)
    bad = to_ref(M.flip_gate(M.gen_multiplier_miter(10, "array", "wallace"), 700), ref)
    for x, want in ((good, "EQUIVALENT"), (bad, "COUNTEREXAMPLE")):
        sm = ref.sweep.SubMiter(circuit=x, origin=(0, 0), merged_history={},
                                pi_map=tuple(range(1, x.num_pis + 1)), id=0)
        r = ref.sched.dispatch(sm, ref.sched.EnginePlan(es_threads=1))
        assert r.verdict == want and r.engine == "es"
        if want == "COUNTEREXAMPLE":
            assert ref.eval.evaluate(x, r.witness) == 1
        # ES on the GPU racing the reference's own SAT engine
        r2 = ref.sched.dispatch(sm, ref.sched.EnginePlan(sat_threads=1, es_threads=1))
        assert r2.verdict == want


def test_reference_programs_run_on_b200(gpu, ref, golden):
    """run_exhaustive on the reference's own InstrProgram objects (the
    SPEC.md:359 seam) equals the reference's golden single-worker results."""
    specs = {s["name"]: s for s in recipes.miter_population()}
    for g in golden["miters"]:
        if g["num_pis"] > 24:
            continue
        x = to_ref(recipes.build_miter_recipe(specs[g["name"]]), ref)
        p = ref.es.compile_program(x)  # the reference's compiler and types
        r = ref.es.run_exhaustive(p)   # patched: the B200 engine
        assert (r.verdict, r.patterns_evaluated) == (g["verdict"], g["patterns_evaluated"]), g["name"]
        if r.witness is not None:
            assert sum(b << i for i, b in enumerate(r.witness)) == g["witness_index"]
