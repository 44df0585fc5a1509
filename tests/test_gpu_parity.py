"""Parity of the CUDA engines with the reference, through the C ABI.

Golden = tests/golden/golden.json, produced by the reference itself
(make_golden.py).  Every verdict, minimum-index witness and
patterns_evaluated must match bit-exactly, for both engines (K1 JIT, K2
interpreter) and for the batched interpreter path.
"""
import pytest

from paper_2512_06627_b200 import es
from tests.golden import recipes

pytestmark = pytest.mark.gpu


def _check(r, g, ctx):
    assert r.verdict == g["verdict"], ctx
    assert r.witness_index == g["witness_index"], ctx
    assert r.patterns_evaluated == g["patterns_evaluated"], ctx


def test_random_population_interp_batch(golden, gpu):
    rows = golden["random"]
    progs = [es.compile_program(recipes.build_random(g)) for g in rows]
    res = es.run_exhaustive_batch(progs)
    for g, r in zip(rows, res):
        _check(r, g, (g["pop"], g["seed"]))


def test_random_population_interp_single(golden, gpu):
    for g in golden["random"][::7]:
        r = es.run_exhaustive(es.compile_program(recipes.build_random(g)), engine="interp")
        _check(r, g, (g["pop"], g["seed"]))


def test_random_population_jit(golden, gpu):
    rows = [g for g in golden["random"] if g["pop"] == "wide"] + golden["random"][:500:25]
    for g in rows:
        r = es.run_exhaustive(es.compile_program(recipes.build_random(g)), engine="jit")
        _check(r, g, (g["pop"], g["seed"]))


@pytest.mark.parametrize("engine", ["jit", "interp"])
def test_miters(golden, gpu, engine):
    specs = {s["name"]: s for s in recipes.miter_population()}
    for g in golden["miters"]:
        if engine == "interp" and (g["num_pis"] > 26 or g["num_registers"] > 400):
            continue
        x = recipes.build_miter_recipe(specs[g["name"]])
        r = es.run_exhaustive(es.compile_program(x), engine=engine)
        _check(r, g, g["name"])


@pytest.mark.parametrize("block", [128, 256, 512])
def test_jit_block_sizes(golden, gpu, block):
    specs = {s["name"]: s for s in recipes.miter_population()}
    for name in ("mult10_array_booth", "mult12_array_wallace_flip1108", "adder5_ripple_lookahead"):
        g = next(q for q in golden["miters"] if q["name"] == name)
        r = es.run_exhaustive(es.compile_program(recipes.build_miter_recipe(specs[name])),
                              engine="jit", block_threads=block)
        _check(r, g, (name, block))


def test_imad_offload_random(golden, gpu):
    """IMAD-mapped LUTs (f(x, word PI)) on random XAGs with many word PIs."""
    for g in golden["random"]:
        if g["pop"] != "wide":
            continue
        r = es.run_exhaustive(es.compile_program(recipes.build_random(g)), engine="jit")
        _check(r, g, g["seed"])
