"""LUT-3 mapping + schedule: the kernel body's CPU model (es_map_eval, same
word layout as K1) must equal the oracle truth table bit for bit."""
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.xag import XagBuilder, random_xag
from tests.golden import recipes


def tt_words(tt: int, n: int) -> np.ndarray:
    nw = 1 << max(n - 5, 0)
    mask = 0xFFFFFFFF if n >= 5 else (1 << (1 << n)) - 1
    return np.array([(tt >> (32 * w)) & mask for w in range(nw)], dtype=np.uint32)


def check(x):
    p = es.compile_program(x)
    got = es.map_eval(p, 0, 1 << max(x.num_pis - 5, 0))
    assert np.array_equal(got, tt_words(O.truth_table(x), x.num_pis))


def test_mapped_random_population(golden):
    for g in golden["random"][::3]:
        if g["num_pis"] <= 20:
            check(recipes.build_random(g))


def test_mapped_random_wide():
    rng = random.Random(5)
    for s in range(60):
        check(random_xag(rng.randint(1, 16), rng.randint(0, 500), 90_000 + s))


@pytest.mark.parametrize("arch", ["diagonal", "wallace", "booth"])
def test_mapped_multiplier_mutants(arch):
    for w in (4, 6, 8):
        m = M.gen_multiplier_miter(w, "array", arch)
        check(m)
        for s in range(4):
            try:
                check(M.mutate(m, s))
            except ValueError:
                pass


def test_mapped_adders_and_edges():
    for w in range(1, 9):
        check(M.gen_adder_miter(w))
    b = XagBuilder(3)
    check(b.finish([b.pi(2)]))             # output is a lane PI
    check(b.finish([~b.pi(3)]))
    b = XagBuilder(9)
    check(b.finish([~b.pi(8)]))            # output is a word PI
    check(b.finish([b.add_and(b.pi(1), b.pi(9))]))
    b = XagBuilder(6)
    g = b.add_xor(b.add_and(b.pi(1), b.pi(2)), b.add_and(b.pi(3), b.pi(4)))  # all lane PIs: folds
    check(b.finish([g]))


def test_mapped_window_offsets():
    """Words far from 0 (high PIs set) evaluate like the oracle's rows."""
    m = M.flip_gate(M.gen_multiplier_miter(12, "array", "wallace"), 1108)
    p = es.compile_program(m)
    words = es.map_eval(p, 8390656 >> 5, 4)
    assert words[0] != 0 and (int(words[0]) & -int(words[0])).bit_length() - 1 == 8390656 & 31


def test_mapping_reduces_issue_count():
    for x in (M.gen_multiplier_miter(12, "array", "wallace"),
              M.gen_multiplier_miter(16, "array", "booth"),
              M.gen_adder_miter(8)):
        st = es.map_stats(es.compile_program(x))
        assert st["luts"] < 0.7 * st["gates"], st
