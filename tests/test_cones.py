"""Config 4: sub-miter extraction (C++ es_batch_extract and the Python
mirror) against the reference's own extract_submiter (golden "cones" rows,
generated with cecprove.sweep.extract_submiter), and the batched device
sweep against the reference's run_exhaustive(workers=1) on those cones."""
import pytest

from paper_2512_06627_b200 import cones, es
from tests.golden import recipes


@pytest.fixture(scope="module")
def round0():
    m, pairs = next(cones.config4_pairs())
    return m, pairs


def test_cpp_extraction_matches_reference(golden, round0):
    m, pairs = round0
    rows = golden["cones"]
    nb = cones.NativeBatch(m, [tuple(r["pair"]) for r in rows])
    assert len(nb) == len(rows)
    for i, g in enumerate(rows):
        sm = nb.submiter(i)
        assert recipes.xag_sha(sm.circuit) == g["xag_sha"], i
        assert list(sm.pi_map) == g["pi_map"]
        inf = nb.info(i)
        assert inf["num_registers"] == g["num_registers"] and inf["G"] == g["G"]
        p = es.compile_program(sm.circuit)
        assert recipes.prog_sha(p.rows(), p.num_registers) == g["prog_sha"]


def test_python_mirror_matches_reference(golden, round0):
    m, _ = round0
    for g in golden["cones"][:60]:
        a, b, pol = g["pair"]
        sm = cones.extract_submiter(m, a, b, polarity=bool(pol))
        assert recipes.xag_sha(sm.circuit) == g["xag_sha"]
        assert list(sm.pi_map) == g["pi_map"]


def test_pairs_are_in_range_and_deterministic(round0):
    m, pairs = round0
    m2, pairs2 = next(cones.config4_pairs())
    assert pairs[:50] == pairs2[:50]
    nb = cones.NativeBatch(m, pairs[:200])
    for i in range(len(nb)):
        assert 14 <= nb.info(i)["num_pis"] <= 24


def test_config4_workload_shape():
    b = cones.config4_batch(1500)
    assert len(b) == 1500
    hs = {b.info(i)["hash"] for i in range(len(b))}
    assert len(hs) == 1500


def test_k2_program_shapes(round0):
    """es_batch_k2_stats: -1 before prepare; afterwards every interpreter
    program fits the launch-group rule of the runtime (<= 176 slots; over 88
    slots, slot file + staged records fit two CTAs per SM at one word per
    thread, unless uncofactored) and the table's gate counts match G."""
    m, pairs = round0
    nb = cones.NativeBatch(m, pairs[:300])
    st = nb.k2_stats()
    assert (st["num_slots"] == -1).all() and (st["num_records"] == -1).all()
    nb.prepare()
    st = nb.k2_stats()
    tab = nb.table()
    for i in range(len(nb)):
        slots, recs, k = int(st["num_slots"][i]), int(st["num_records"][i]), int(st["cofactor_pis"][i])
        assert slots >= tab["num_pis"][i] and 0 <= k <= 6
        assert recs >= (tab["G"][i] > 0)  # gates + one OUT record per copy
        if k > 0:
            assert slots <= 176
            assert slots <= 88 or slots * 512 + (recs + 1) * 16 <= 115600
        assert tab["G"][i] == nb.info(i)["G"]


def test_merges_collapse_nodes(round0):
    """A merge map (proven node -> earlier representative) is honoured like
    sweep.py:84-89: extracting (a, b) with the later node merged onto the
    earlier one is constant; a cyclic map fails loudly, not by crashing."""
    from paper_2512_06627_b200 import _native as N
    from paper_2512_06627_b200.xag import Lit
    m, pairs = round0
    a, b, pol = pairs[0]
    lo, hi = min(a, b), max(a, b)
    nb = cones.NativeBatch(m, [(a, b, pol)], merges={hi: Lit(lo, pol)})
    sm = nb.submiter(0)
    py = cones.extract_submiter(m, a, b, merges={hi: Lit(lo, pol)}, polarity=pol)
    assert recipes.xag_sha(sm.circuit) == recipes.xag_sha(py.circuit)
    assert sm.circuit.outputs[0].node == 0
    # other pairs keep extracting identically under a merge map
    extra = pairs[1:40]
    nb = cones.NativeBatch(m, extra, merges={hi: Lit(lo, pol)})
    for i, (x, y, q) in enumerate(extra):
        try:
            py = cones.extract_submiter(m, x, y, merges={hi: Lit(lo, pol)}, polarity=q)
        except KeyError:
            continue
        assert recipes.xag_sha(nb.submiter(i).circuit) == recipes.xag_sha(py.circuit)


@pytest.mark.gpu
def test_batched_sweep_matches_reference(golden, round0, gpu):
    m, _ = round0
    rows = golden["cones"]
    nb = cones.NativeBatch(m, [tuple(r["pair"]) for r in rows])
    res = nb.run()
    for g, r in zip(rows, res):
        assert r.verdict == g["verdict"]
        assert r.witness_index == g["witness_index"]
        assert r.patterns_evaluated == g["patterns_evaluated"]


@pytest.mark.gpu
def test_config4_batch_vs_single_runs(gpu):
    b = cones.config4_batch(600)
    res = b.run()
    for i in range(0, 600, 20):
        sm = b.submiter(i)
        r = es.run_exhaustive(es.compile_program(sm.circuit), engine="jit")
        assert (r.verdict, r.witness_index) == (res[i].verdict, res[i].witness_index), i


def test_sweep_round_batch_shape():
    """The EQ-heavy config-4 variant's cones: distinct, 14-24 PIs, from the
    configs[2] miter's own 64-word candidate classes."""
    import numpy as np

    from paper_2512_06627_b200 import cones

    b = cones.sweep_round_batch()
    tab = b.table()
    assert len(b) > 100
    assert tab["num_pis"].min() >= 14 and tab["num_pis"].max() <= 24
    assert len(np.unique(tab["hash"])) == len(b)
