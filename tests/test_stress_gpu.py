"""Randomised parity on the GPU (a short run of scripts/stress_parity.py):
every engine and cofactor / build policy (direct SASS included) returns the oracle's
canonical minimum-index witness on fault miters with deep witnesses."""
import importlib.util
import os

import pytest

from oracle import oracle as O
from paper_2512_06627_b200 import es

pytestmark = pytest.mark.gpu

_spec = importlib.util.spec_from_file_location(
    "stress_parity", os.path.join(os.path.dirname(__file__), "..", "scripts", "stress_parity.py"))
SP = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(SP)


@pytest.mark.parametrize("seed", [11, 12])
def test_random_fault_miters_all_engines(gpu, seed):
    n_neq = 0
    for name, x in SP.cases(40, seed):
        _, ref_w, _ = O.min_witness(O.compile_program(x))
        n_neq += ref_w is not None
        p = es.compile_program(x)
        for engine, cof, parts in SP.MODES:  # (direct-SASS builds first: jit_parts -1)
            r = es.run_exhaustive(p, engine=engine, cofactor=cof, jit_parts=parts)
            assert r.witness_index == ref_w, (name, x.num_pis, engine, cof, parts, r.witness_index, ref_w)
    assert n_neq > 0
