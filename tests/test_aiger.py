"""AIGER ingest + XOR recovery (csrc/es_aiger.cpp) against
fixtures the reference generated (tests/golden/make_golden_aiger.py): the
written bytes, the parsed circuit (ASCII, shuffled ASCII, binary), the
XOR-recovered circuit and its ES program size, and every error class."""
import hashlib
import json
import os

import pytest

from paper_2512_06627_b200 import aiger as A
from paper_2512_06627_b200 import es
from tests.golden import recipes

GOLD = os.path.join(os.path.dirname(__file__), "golden", "aiger_golden.json")


@pytest.fixture(scope="module")
def gold():
    return json.load(open(GOLD))


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:24]


def test_roundtrip_matches_reference(gold):
    for k, row in enumerate(gold["rows"]):
        x = recipes.build_aiger_circuit(row)
        assert recipes.xag_sha(x) == row["xag_sha"]
        text = A.write_aiger(x)
        assert sha(text) == row["aag_sha"], row
        parsed = A.parse_aiger(text)
        assert recipes.xag_sha(parsed) == row["parsed_sha"], row
        assert recipes.xag_sha(A.parse_aiger(recipes.to_binary_aiger(text))) == row["binary_sha"], row
        if "shuffled_sha" in row:
            assert recipes.xag_sha(A.parse_aiger(recipes.shuffled_ascii(text, k))) == row["shuffled_sha"]
        rec = A.detect_xors(parsed)
        assert recipes.xag_sha(rec) == row["xors_sha"], row
        if "G" in row:
            assert es.compile_program(rec).num_gates == row["G"]


def test_error_classes_match_reference(gold):
    names = {"MalformedHeader": A.MalformedHeader, "LatchesUnsupported": A.LatchesUnsupported,
             "DanglingLiteral": A.DanglingLiteral, "AigerError": A.AigerError}
    for case in gold["errors"]:
        data = bytes.fromhex(case["hex"])
        if case["error"] is None:
            A.parse_aiger(data)
            continue
        with pytest.raises(names[case["error"]]) as ei:
            A.parse_aiger(data)
        assert type(ei.value).__name__ == case["error"], data


def test_load_circuit_recovers_the_miter(tmp_path):
    """cli._load_circuit: a written XAG miter comes back with its XORs, and
    its ES program is the original's (same G)."""
    from paper_2512_06627_b200 import miter as M
    m = M.gen_multiplier_miter(8, "array", "booth")
    path = tmp_path / "m.aag"
    path.write_bytes(A.write_aiger(m))
    back = A.load_circuit(str(path))
    assert es.compile_program(back).num_gates == es.compile_program(m).num_gates


@pytest.mark.gpu
def test_aiger_to_verdict(gpu, golden, tmp_path):
    """End to end: AIGER file -> load_circuit -> es_check on the GPU gives the
    reference's verdict and minimum-index witness (golden miters)."""
    specs = {s["name"]: s for s in recipes.miter_population()}
    for name in ("mult12_array_wallace", "mult12_array_wallace_flip1108", "mult10_array_booth"):
        g = next(q for q in golden["miters"] if q["name"] == name)
        x = recipes.build_miter_recipe(specs[name])
        path = tmp_path / f"{name}.aag"
        path.write_bytes(A.write_aiger(x))
        back = A.load_circuit(str(path))
        r = es.run_exhaustive(es.compile_program(back))
        assert r.verdict == g["verdict"] and r.witness_index == g["witness_index"], name
