"""K2 interpreter programs (es_k2prog.cpp): the CPU model of the interpreter
(16-byte records, accumulator forwarding, OUT records per cofactor copy) must
equal the oracle truth table bit for bit -- for the depth K2 picks itself and
for every forced cofactor depth."""
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200._native import NativeError
from paper_2512_06627_b200.xag import XagBuilder, random_xag
from tests.golden import recipes
from tests.test_mapper import tt_words


def check(x, ks=(0, 1, 2, 3, 4, 5, 6)):
    p = es.compile_program(x)
    n = x.num_pis
    want = tt_words(O.truth_table(x), n)
    nw = 1 << max(n - 5, 0)
    assert np.array_equal(es.k2_eval(p, 0, nw), want), (n, "auto")
    for k in ks:
        if k > n - 5:
            continue
        try:
            got = es.k2_eval(p, 0, nw, k=k)
        except NativeError as e:   # fewer word PIs in the cone than k
            assert e.code == -4
            continue
        assert np.array_equal(got, want), (n, k)


def test_k2_random_population(golden):
    for g in golden["random"][::5]:
        if g["num_pis"] <= 18:
            check(recipes.build_random(g), ks=(0, 2))


def test_k2_random_wide():
    rng = random.Random(17)
    for s in range(40):
        check(random_xag(rng.randint(6, 15), rng.randint(1, 400), 50_000 + s))


@pytest.mark.parametrize("arch", ["diagonal", "wallace", "booth"])
def test_k2_multipliers_and_mutants(arch):
    for w in (4, 6, 8):
        m = M.gen_multiplier_miter(w, "array", arch)
        check(m)
        for s in range(3):
            try:
                check(M.mutate(m, s))
            except ValueError:
                pass


def test_k2_edges():
    for w in (1, 3, 8):
        check(M.gen_adder_miter(w))
    b = XagBuilder(3)
    check(b.finish([b.pi(2)]))                     # output is a lane PI
    b = XagBuilder(9)
    check(b.finish([~b.pi(8)]))                    # output is a (cofactor-able) word PI
    b = XagBuilder(8)                              # copies whose output folds to 0 / 1
    check(b.finish([b.add_and(b.pi(8), b.add_xor(b.pi(7), b.pi(6)))]))
    b = XagBuilder(8)
    check(b.finish([b.add_or(b.pi(8), b.pi(7))]))
    b = XagBuilder(7)
    x = b.add_and(b.pi(6), b.pi(7))
    check(b.finish([b.add_and(x, x)]))


def test_k2_picks_cofactors_on_cones():
    from paper_2512_06627_b200 import cones
    b = cones.config4_batch(300)
    deep = 0
    for i in range(0, len(b), 10):
        sm = b.submiter(i)
        p = es.compile_program(sm.circuit)
        k = es.k2_cofactor_pis(p)
        assert 0 <= k <= 6
        deep += k >= 3
        if sm.circuit.num_pis <= 18:
            check(sm.circuit, ks=(k,))
    assert deep > 0
