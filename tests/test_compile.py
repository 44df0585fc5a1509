"""The product's host compiler against the reference (CPU only).

compile_program must be instruction-for-instruction the reference schedule
(es.py:87-163): the golden fingerprints come from the reference itself.
Also replays the compile-side tests of the reference's test_es.py.
"""
import pytest

from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.xag import XagBuilder
from tests.golden import recipes


def test_compile_matches_reference_random(golden):
    for g in golden["random"]:
        p = es.compile_program(recipes.build_random(g))
        assert recipes.prog_sha(p.rows(), p.num_registers) == g["prog_sha"], (g["pop"], g["seed"])
        assert len(p) == g["num_instrs"] and p.num_gates == g["G"]


def test_compile_matches_reference_miters(golden):
    specs = {s["name"]: s for s in recipes.miter_population()}
    for g in golden["miters"]:
        x = recipes.build_miter_recipe(specs[g["name"]])
        assert recipes.xag_sha(x) == g["xag_sha"], g["name"]
        p = es.compile_program(x)
        assert recipes.prog_sha(p.rows(), p.num_registers) == g["prog_sha"], g["name"]
        assert p.num_registers == g["num_registers"], g["name"]
        if "program" in g:
            assert p.rows() == g["program"]


def test_compile_register_reuse():  # test_es.py:19-30
    b = XagBuilder(8)
    acc = b.pi(1)
    for i in range(2, 9):
        acc = b.add_and(acc, b.pi(i))
    p = es.compile_program(b.finish([acc]))
    assert p.num_registers <= 3
    kinds = [i.op for i in p.instrs]
    assert kinds.count(es.OP_LOAD_PI) == 8
    assert kinds.count(es.OP_AND) == 7
    assert kinds[-1] == es.OP_OUTPUT


def test_compile_rejects_oversized_inputs():  # test_es.py:33-37
    b = XagBuilder(41)
    o = b.add_and(b.pi(1), b.pi(2))
    with pytest.raises(es.TooManyInputs):
        es.compile_program(b.finish([o]))


def test_es_check_ineligible():  # test_es.py:99-103 (never reaches the GPU)
    b = XagBuilder(41)
    o = b.add_and(b.pi(1), b.pi(41))

    class SM:
        circuit = b.finish([o])
    r = es.es_check(SM())
    assert r.verdict == "UNKNOWN" and r.reason == "ineligible" and r.engine == "es"


def test_es_check_budget_zero():  # test_es.py:106-109: timeout before any work
    class SM:
        circuit = M.gen_multiplier_miter(11, "array", "diagonal")
    r = es.es_check(SM(), budget=0.0)
    assert r.verdict == "UNKNOWN" and r.reason == "timeout"


def test_register_compression():  # test_es.py:112-116, test_acceptance.py:150-158
    ratios = []
    for n in (4, 6, 8):
        m = M.gen_multiplier_miter(n, "array", "diagonal")
        ratios.append(es.compile_program(m).num_registers / m.num_gates)
    assert ratios[0] >= ratios[1] >= ratios[2] and ratios[2] <= 0.15
    m = M.gen_multiplier_miter(6, "array", "diagonal")
    assert es.compile_program(m).num_registers / m.num_gates < 0.2


def test_constant_programs():
    b = XagBuilder(3)
    p = es.compile_program(b.finish([b.add_and(b.pi(1), ~b.pi(1))]))
    assert p.rows() == [[3, 0, -1, 0, -1, 0, 0]] and p.num_registers == 0
    p = es.compile_program(b.finish([~b.pi(2)]))
    assert p.rows() == [[0, 0, -1, 0, -1, 0, 2], [3, 0, 0, 1, -1, 0, 0]]


def test_program_dump_and_roundtrip():
    p = es.compile_program(M.gen_multiplier_miter(3, "array", "diagonal"))
    text = p.dump()
    assert text.splitlines()[0].startswith("r0 = load pi")
    assert text.splitlines()[-1].startswith("out ")
    q = es.InstrProgram.from_instrs(p.instrs, p.num_registers, p.num_pis)
    assert q == p


def test_programs_from_reference_objects_are_accepted():
    """run_exhaustive takes the reference's InstrProgram (duck-typed)."""
    p = es.compile_program(M.gen_multiplier_miter(3, "array", "diagonal"))

    class RefLike:
        instrs = p.instrs
        num_registers = p.num_registers
        num_pis = p.num_pis
    assert es.as_program(RefLike()) == p


def test_native_witness_recheck_matches_evaluate():
    """es_xag_eval (the es_check witness re-check, es.py:360-361) equals the
    direct evaluation (eval.py:22-36) on random XAGs and patterns."""
    import random as _r

    from paper_2512_06627_b200 import es as _es
    from paper_2512_06627_b200.miter import evaluate as _ev
    from paper_2512_06627_b200.xag import random_xag as _rx

    rng = _r.Random(7)
    for k in range(60):
        x = _rx(rng.randint(1, 40), rng.randint(0, 300), seed=k)
        for _ in range(8):
            bits = tuple(rng.randint(0, 1) for _ in range(x.num_pis))
            assert _es._recheck(x, bits) == _ev(x, bits)
