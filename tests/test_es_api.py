"""The reference's ES test-suite semantics (pkg/tests/test_es.py:19-116 and
the ES rows of test_acceptance.py), replayed against this engine on the GPU,
plus budget / cancel / session / sharded-sweep behaviour."""
import threading
import time

import pytest

from oracle import oracle as O
from paper_2512_06627_b200 import es, shard
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.verdict import COUNTEREXAMPLE, EQUIVALENT, UNKNOWN
from paper_2512_06627_b200.xag import XagBuilder, random_xag

pytestmark = pytest.mark.gpu


class SM:  # SubMiter stand-in (sweep.py:44-51)
    def __init__(self, x):
        self.circuit = x
        self.origin = (0, 0)
        self.merged_history = {}
        self.pi_map = tuple(range(1, x.num_pis + 1))


def test_exhaustive_zero_on_constant_false_cone(gpu):  # test_es.py:40-45
    b = XagBuilder(4)
    g = b.add_and(b.pi(1), ~b.pi(1))
    r = es.run_exhaustive(es.compile_program(b.finish([g])))
    assert r.verdict == es.EXHAUSTED_ZERO and r.patterns_evaluated == 16


def test_constant_true_rail(gpu):  # es.py:265-270
    b = XagBuilder(5)
    r = es.run_exhaustive(es.compile_program(b.finish([~b.add_and(b.pi(1), ~b.pi(1))])))
    assert r.verdict == es.ES_COUNTEREXAMPLE and r.witness == (0,) * 5
    assert r.patterns_evaluated == 0


def test_counterexample_with_witness(gpu):  # test_es.py:48-55
    b = XagBuilder(4)
    g = b.add_and(b.add_and(b.pi(1), b.pi(2)), b.add_and(b.pi(3), b.pi(4)))
    x = b.finish([g])
    r = es.run_exhaustive(es.compile_program(x))
    assert r.verdict == es.ES_COUNTEREXAMPLE and M.evaluate(x, r.witness) == 1
    assert r.witness == (1, 1, 1, 1)


@pytest.mark.parametrize("engine", ["jit", "interp"])
def test_matches_truth_table(gpu, engine):  # test_es.py:58-67, all 301 seeds
    for seed in range(0, 301, 3 if engine == "jit" else 1):
        x = random_xag(6, 40, seed)
        r = es.run_exhaustive(es.compile_program(x), engine=engine)
        first = O.first_one_row(O.truth_table(x))
        if first is None:
            assert r.verdict == es.EXHAUSTED_ZERO
        else:
            assert r.verdict == es.ES_COUNTEREXAMPLE and r.witness_index == first


def test_workers_agree_on_verdict_and_witness(gpu):  # test_es.py:70-78
    for seed in range(0, 101, 5):
        x = random_xag(7, 50, seed)
        p = es.compile_program(x)
        a = es.run_exhaustive(p, workers=1)
        for w in (2, 3, 4):
            b = es.run_exhaustive(p, workers=w)
            assert (a.verdict, a.witness) == (b.verdict, b.witness)  # stronger than the ref


def test_es_check_equivalent(gpu):  # test_es.py:81-86
    m = M.gen_multiplier_miter(3, "array", "diagonal")
    r = es.es_check(SM(m))
    assert r.verdict == EQUIVALENT and r.engine == "es"
    assert r.stats["patterns"] == 1 << m.num_pis


def test_es_check_counterexample(gpu):  # test_es.py:89-96
    a = random_xag(6, 40, seed=2)
    m = M.build_miter(a, M.mutate(a, seed=4))
    r = es.es_check(SM(m))
    assert r.verdict == COUNTEREXAMPLE and M.evaluate(m, r.witness) == 1


def test_oracle_agreement_500(gpu, golden):  # test_acceptance.py:82-101 (ES column)
    for g in golden["random"][:500]:
        x = random_xag(g["n_pis"], g["n_gates"], g["seed"])
        r = es.es_check(SM(x), workers=1, engine="interp")
        assert r.verdict != UNKNOWN
        assert (r.verdict == EQUIVALENT) == (g["witness_index"] is None)
        if r.verdict == COUNTEREXAMPLE:
            assert M.evaluate(x, r.witness) == 1


def test_budget_timeout_midway(gpu):
    m = M.gen_multiplier_miter(16, "array", "booth")
    p = es.compile_program(m)
    # one word per iteration (no cofactor copies): a ~10 ms sweep, so a 4 ms
    # budget must stop it midway
    es.run_exhaustive(p, engine="jit", cofactor="none")  # warm the JIT cache
    r = es.run_exhaustive(p, engine="jit", budget=0.004, slice_ms=1.0, cofactor="none")
    assert r.verdict == es.BUDGET_EXCEEDED
    assert 0 < r.patterns_evaluated < 1 << 32
    c = es.es_check(SM(m), budget=0.004, cofactor="none")
    assert c.verdict == UNKNOWN and c.reason == "timeout"


def test_cancel(gpu):
    m = M.gen_multiplier_miter(16, "array", "booth")
    ev = threading.Event()
    threading.Timer(0.003, ev.set).start()
    es.run_exhaustive(es.compile_program(m), engine="jit")  # warm JIT
    t = time.monotonic()
    c = es.es_check(SM(m), cancel=ev.is_set)
    if c.verdict == UNKNOWN:
        assert c.reason == "cancelled"
    assert time.monotonic() - t < 5
    ev2 = threading.Event()
    ev2.set()
    c = es.es_check(SM(m), cancel=ev2.is_set)
    assert c.verdict == UNKNOWN and c.reason == "cancelled"


def test_session_and_single_rank_sharded_sweep(gpu, golden):
    import torch
    for name in ("mult12_array_wallace", "mult12_array_wallace_flip1108",
                 "mult14_array_diagonal"):
        g = next(q for q in golden["miters"] if q["name"] == name)
        from tests.golden import recipes
        spec = next(s for s in recipes.miter_population() if s["name"] == name)
        p = es.compile_program(recipes.build_miter_recipe(spec))
        for slices in (1, 3):
            r = shard.sweep_sharded(p, device=0, slices=slices)
            assert (r.verdict, r.witness_index, r.patterns_evaluated) == (
                g["verdict"], g["witness_index"], g["patterns_evaluated"]), name
        # emulate 3 ranks on one GPU: disjoint residue classes, shared minimum
        s = shard.session_for(p, 0)
        best = torch.full((1,), 1 << p.num_pis, dtype=torch.int64, device="cuda:0")
        st = torch.cuda.current_stream().cuda_stream
        for rank in range(3):
            s.launch(st, best.data_ptr(), 0, s.n_chunks, rank, 3)
        b = int(best.item())
        assert (None if b >= 1 << p.num_pis else b) == g["witness_index"], name


def test_batch_api(gpu, golden):
    from tests.golden import recipes
    rows = golden["random"][:200]
    res = es.es_check_batch([SM(recipes.build_random(g)) for g in rows])
    for g, r in zip(rows, res):
        assert (r.verdict == EQUIVALENT) == (g["witness_index"] is None)
        if r.verdict == COUNTEREXAMPLE:
            assert sum(b << i for i, b in enumerate(r.witness)) == g["witness_index"]


def test_alu_peak_positive(gpu):
    v, ms = shard.alu_peak(0)
    assert v > 1e12 and ms > 0
