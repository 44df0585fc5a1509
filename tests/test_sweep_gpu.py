"""The sweep with the ES engine on the GPU (paper_2512_06627_b200.sweep,
SURVEY 8(f) next-1) against the reference's own sweep(engine="es") results
(tests/golden/make_golden_sweep.py): same verdict on every miter; the same
witness where it is canonical -- refuted by the shared random simulation, or
a single failing pattern found by the final ES obligation."""
import json
import os

import pytest

from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.sweep import SweepConfig, sweep
from tests.golden import recipes

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "sweep_golden.json")


def test_sweep_matches_reference(gpu):
    rows = json.load(open(GOLD))["rows"]
    for row in rows:
        x = recipes.build_sweep_circuit(row)
        assert recipes.xag_sha(x) == row["xag_sha"]
        r = sweep(x, SweepConfig())
        assert r.verdict == row["verdict"], row
        if r.verdict == "COUNTEREXAMPLE":
            assert M.evaluate(x, r.witness) == 1
            if row["engine"] == "sim" or "needle" in row:
                assert list(r.witness) == row["witness"], row
        if row["verdict"] == "EQUIVALENT":
            assert r.stats["merges"] + r.stats["structural_merges"] > 0
