"""Config circuits: the new generators compute the right functions, and the
reference-equivalent ones are gate-for-gate the reference's (golden xag_sha)."""
import itertools

import pytest

from paper_2512_06627_b200 import miter as M


def eval_all(x, bits):
    vals = [0] * (1 + x.num_pis + len(x.gates))
    for i, v in enumerate(bits):
        vals[1 + i] = v
    for i, g in enumerate(x.gates):
        a = vals[g.in0.node] ^ int(g.in0.neg)
        b = vals[g.in1.node] ^ int(g.in1.neg)
        vals[1 + x.num_pis + i] = (a & b) if g.kind == 0 else (a ^ b)
    return sum((vals[o.node] ^ int(o.neg)) << k for k, o in enumerate(x.outputs))


@pytest.mark.parametrize("arch", ["array", "diagonal", "wallace", "booth"])
@pytest.mark.parametrize("w", [2, 4, 6])
def test_multipliers_multiply(arch, w):
    x = M.gen_multiplier(w, arch)
    for a, b in itertools.product(range(1 << w), repeat=2):
        bits = [(a >> i) & 1 for i in range(w)] + [(b >> i) & 1 for i in range(w)]
        assert eval_all(x, bits) == a * b


@pytest.mark.parametrize("arch", ["ripple", "lookahead"])
@pytest.mark.parametrize("w", [1, 3, 5, 8])
def test_adders_add(arch, w):
    x = M.gen_adder(w, arch)
    for a, b in itertools.product(range(1 << w), repeat=2):
        bits = [(a >> i) & 1 for i in range(w)] + [(b >> i) & 1 for i in range(w)]
        assert eval_all(x, bits) == a + b


def test_config_miters_shape():
    a8 = M.gen_adder_miter(8)
    assert a8.num_pis == 16 and len(a8.outputs) == 1
    assert M.gen_multiplier_miter(12, "array", "wallace").num_pis == 24
    assert M.gen_multiplier_miter(16, "array", "booth").num_pis == 32
    assert M.truth_table(a8) == 0


def test_booth_rejects_odd_width():
    with pytest.raises(M.WidthOutOfRange):
        M.gen_multiplier(5, "booth")
