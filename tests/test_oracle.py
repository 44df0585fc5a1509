"""Pin the CPU oracle (oracle/) to the reference's own outputs.

tests/golden/golden.json was produced by the reference package itself
(make_golden.py imports cecprove): compile_program fingerprints and
run_exhaustive(workers=1) verdict / witness / patterns_evaluated.  The oracle
must reproduce every row before it may judge the GPU path.
"""
import pytest

from oracle import oracle as O
from tests.golden import recipes


def _rows(p):
    return [[int(v) for v in r] for r in p.rows()]


def test_golden_population_sizes(golden):
    assert len(golden["random"]) == 500 + 301 + 101 + 60
    assert len(golden["miters"]) >= 70


def test_oracle_compile_matches_reference_random(golden):
    for g in golden["random"]:
        x = recipes.build_random(g)
        assert recipes.xag_sha(x) == g["xag_sha"], (g["pop"], g["seed"])
        p = O.compile_program(x)
        assert recipes.prog_sha(_rows(p), p.num_registers) == g["prog_sha"], (g["pop"], g["seed"])
        assert p.num_gate_instrs == g["G"]


def test_oracle_run_matches_reference_random(golden):
    for g in golden["random"]:
        x = recipes.build_random(g)
        r = O.run_exhaustive(O.compile_program(x), workers=1)
        assert r.verdict == g["verdict"], (g["pop"], g["seed"])
        assert r.witness_index == g["witness_index"], (g["pop"], g["seed"])
        assert r.patterns_evaluated == g["patterns_evaluated"], (g["pop"], g["seed"])


def test_oracle_truth_table_and_evaluate(golden):
    for g in golden["random"][:300]:
        x = recipes.build_random(g)
        first = O.first_one_row(O.truth_table(x))
        assert first == g["witness_index"]
        if first is not None:
            bits = [(first >> i) & 1 for i in range(x.num_pis)]
            assert O.evaluate(x, bits) == 1


def test_oracle_miters(golden):
    specs = {s["name"]: s for s in recipes.miter_population()}
    for g in golden["miters"]:
        x = recipes.build_miter_recipe(specs[g["name"]])
        assert recipes.xag_sha(x) == g["xag_sha"], g["name"]
        p = O.compile_program(x)
        assert recipes.prog_sha(_rows(p), p.num_registers) == g["prog_sha"], g["name"]
        assert p.num_registers == g["num_registers"]
        if g["num_pis"] <= 24:
            r = O.run_exhaustive(p, workers=1)
            assert (r.verdict, r.witness_index, r.patterns_evaluated) == (
                g["verdict"], g["witness_index"], g["patterns_evaluated"]), g["name"]


def test_oracle_full_program_rows(golden):
    rows = [g for g in golden["miters"] if "program" in g]
    assert rows
    specs = {s["name"]: s for s in recipes.miter_population()}
    for g in rows:
        p = O.compile_program(recipes.build_miter_recipe(specs[g["name"]]))
        assert _rows(p) == g["program"]


@pytest.mark.slow
def test_oracle_min_witness_deep_faults(golden):
    """Multi-threaded minimum-index sweep == reference workers=1 witness on
    the 28-31-bit-deep 16x16 faults (the config-5 fixtures)."""
    specs = {s["name"]: s for s in recipes.miter_population()}
    for g in golden["miters"]:
        if "flip_gate" not in g or g["num_pis"] != 32 or g["witness_index"] > 1 << 29:
            continue
        p = O.compile_program(recipes.build_miter_recipe(specs[g["name"]]))
        v, idx, _ = O.min_witness(p)
        assert (v, idx) == (g["verdict"], g["witness_index"]), g["name"]


def test_oracle_workers_verdict_invariant(golden):
    for g in golden["random"][500:560]:
        p = O.compile_program(recipes.build_random(g))
        for w in (2, 3, 8):
            r = O.run_exhaustive(p, workers=w)
            assert r.verdict == g["verdict"]


def test_oracle_budget_zero():
    from paper_2512_06627_b200 import miter as M
    p = O.compile_program(M.gen_multiplier_miter(11, "array", "diagonal"))
    assert O.run_exhaustive(p, budget=0.0).verdict == O.BUDGET_EXCEEDED
