"""Cofactor expansion of K1 (es_cofactor.cpp): with k word PIs fixed per copy,
the kernel body's CPU model must still equal the oracle truth table bit for
bit, for every k, and the PTX must compile without a GPU."""
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200._native import NativeError
from paper_2512_06627_b200.xag import XagBuilder, random_xag
from tests.test_mapper import tt_words


def check_all_k(x, ks=(1, 2, 3, 4)):
    p = es.compile_program(x)
    n = x.num_pis
    want = tt_words(O.truth_table(x), n)
    for k in ks:
        if k > n - 5:
            continue
        try:
            got = es.map_eval(p, 0, 1 << (n - 5), k=k)
        except NativeError as e:  # fewer word PIs in the cone than k
            assert e.code == -4
            continue
        assert np.array_equal(got, want), (n, k)


def test_cofactor_random():
    rng = random.Random(11)
    for s in range(40):
        check_all_k(random_xag(rng.randint(7, 14), rng.randint(1, 400), 70_000 + s))


@pytest.mark.parametrize("arch", ["diagonal", "wallace", "booth"])
def test_cofactor_multipliers_and_mutants(arch):
    for w in (4, 6, 8):
        m = M.gen_multiplier_miter(w, "array", arch)
        check_all_k(m)
        for s in range(3):
            try:
                check_all_k(M.mutate(m, s))
            except ValueError:
                pass


def test_cofactor_edges():
    for w in (4, 6, 8):
        check_all_k(M.gen_adder_miter(w))
    b = XagBuilder(9)
    check_all_k(b.finish([~b.pi(8)]))             # output is a cofactor-able word PI
    b = XagBuilder(9)
    check_all_k(b.finish([b.add_and(b.pi(9), b.add_and(b.pi(8), b.pi(1)))]))
    b = XagBuilder(8)                              # copies whose output folds to a constant
    check_all_k(b.finish([b.add_and(b.pi(8), b.add_xor(b.pi(7), b.pi(6)))]))
    b = XagBuilder(8)
    check_all_k(b.finish([b.add_or(b.pi(8), b.pi(7))]))


def test_cofactor_pis_pick_smallest_fanout():
    m = M.gen_multiplier_miter(16, "array", "booth")
    p = es.compile_program(m)
    st = [es.map_stats(p, k) for k in range(5)]
    assert st[1]["cofactor_pis"] == [32]
    assert st[3]["cofactor_pis"] == [30, 31, 32]
    per_word = [s["luts"] / 2 ** k for k, s in enumerate(st)]
    assert per_word[3] < 0.3 * per_word[0]        # 8 words for < 2.4x the LUTs of one
    assert all(a > b for a, b in zip(per_word, per_word[1:]))


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_cofactor_ptx_compiles(k):
    m = M.gen_multiplier_miter(8, "array", "booth")
    r = es.jit_check(es.compile_program(m), 256, k=k)
    assert r["cubin_bytes"] > 0 and r["spill_bytes"] == 0


@pytest.mark.parametrize("k,copies", [(2, 1), (2, 3), (3, 5), (4, 6), (4, 11)])
def test_restricted_copies_model(k, copies):
    """The second phase's restricted variant (copies 0..copies-1 of the same
    cofactor set): words of those copies equal the full variant's, the other
    copies' words are 0 (not evaluated), and the body is smaller."""
    x = M.gen_multiplier_miter(6, "array", "booth")
    bad = M.flip_gate(x, 40)
    for c in (x, bad):
        p = es.compile_program(c)
        n = c.num_pis
        full = es.map_eval(p, 0, 1 << (n - 5), k=k)
        part = es.map_eval_restricted(p, 0, 1 << (n - 5), k, copies)
        cof = es.map_stats(p, k)["cofactor_pis"]
        w = np.arange(1 << (n - 5), dtype=np.uint64)
        copy = np.zeros_like(w)
        for b, j in enumerate(cof):
            copy |= ((w >> np.uint64(j - 6)) & np.uint64(1)) << np.uint64(b)
        keep = copy < copies
        assert np.array_equal(part[keep], full[keep])
        assert not part[~keep].any()
    assert es.map_stats_restricted(p, k, copies)["luts"] < es.map_stats(p, k)["luts"]
