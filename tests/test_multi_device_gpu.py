"""One es_run over several devices (es_run_opts.devices; SURVEY 8(b)
``es_run(prog, n_gpus, ...)``, the reference's workers as GPUs,
es.py:272-331) and the two-phase non-equivalent search.

The box has one B200, so "several devices" are several host threads on
device 0 (devices=[0, 0, ...]): every thread drives its own stream and
residue class of chunks, and they share one minimum word -- the same code
path as distinct GPUs with peer access, minus NVLink.  Every verdict,
minimum-index witness and patterns_evaluated must equal the reference's
single-worker run (tests/golden/golden.json)."""
import pytest

from paper_2512_06627_b200 import es
from tests.golden import recipes

pytestmark = pytest.mark.gpu

DEEP = ["mult16_array_booth_flip2204", "mult16_array_booth_flip1953", "mult16_array_booth_flip1406",
        "mult16_array_booth_flip1882", "mult16_array_booth_flip1220", "mult16_array_booth",
        "mult12_array_wallace_flip1108", "mult14_array_booth", "adder8_ripple_lookahead"]


@pytest.fixture(scope="module")
def miters(golden):
    specs = {s["name"]: s for s in recipes.miter_population()}
    rows = {g["name"]: g for g in golden["miters"]}
    return {n: (es.compile_program(recipes.build_miter_recipe(specs[n])), rows[n]) for n in DEEP}


def _check(r, g, ctx):
    assert (r.verdict, r.witness_index, r.patterns_evaluated) == \
        (g["verdict"], g["witness_index"], g["patterns_evaluated"]), ctx


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0]])
@pytest.mark.parametrize("cof", ["throughput", "none", 2])
def test_multi_device_parity(gpu, miters, devices, cof):
    for name, (p, g) in miters.items():
        r = es.run_exhaustive(p, engine="jit", cofactor=cof, devices=devices)
        _check(r, g, (name, devices, cof))
        assert r.stats["n_devices"] == len(devices)
        assert r.stats["witness_minimal"] or r.verdict != es.ES_COUNTEREXAMPLE


def test_neq_two_phase_sweeps_below_the_witness(gpu, miters):
    """Config 5: the cheapest cofactor PIs are the top pattern bits, so a
    witness above 2^28 needs the second phase; it must sweep little more than
    the space below the witness, not the whole space."""
    p, g = miters["mult16_array_booth_flip1953"]
    for devices in (None, [0, 0]):
        r = es.run_exhaustive(p, engine="jit", cofactor="throughput", devices=devices)
        _check(r, g, devices)
        assert r.stats["cofactor_pis"] == 4 and r.stats["phases"] == 2
        assert r.stats["patterns_swept"] < 0.5 * (1 << 32), r.stats


def test_neq_shallow_witness_single_phase(gpu):
    """A witness below 2^28 (its cofactor bits all 0) is proven by phase 1."""
    needle = (1 << 24) + 5
    x = recipes.build_sweep_circuit({"kind": "mult", "width": 16, "a": "array", "b": "booth",
                                     "needle": needle})
    r = es.run_exhaustive(es.compile_program(x), engine="jit", cofactor="throughput")
    assert r.witness_index == needle and r.stats["phases"] == 1
    assert r.stats["patterns_swept"] < (1 << 30)


@pytest.mark.parametrize("needle", [(1 << 28) + 1, 3 << 29, (1 << 31) + 12345, (1 << 32) - 1])
def test_neq_deep_needles(gpu, needle):
    """A single failing pattern at any depth is found exactly, whichever
    second phase the policy picks (restricted copies, low cofactor set, or
    finishing the first sweep), on one device or two host threads."""
    x = recipes.build_sweep_circuit({"kind": "mult", "width": 16, "a": "array", "b": "booth",
                                     "needle": needle})
    p = es.compile_program(x)
    for devices in (None, [0, 0]):
        r = es.run_exhaustive(p, engine="jit", cofactor="throughput", devices=devices)
        assert (r.verdict, r.witness_index) == (es.ES_COUNTEREXAMPLE, needle), (devices, r.stats)
        assert r.patterns_evaluated == ((needle >> 14) + 1) << 14


def test_devices_all_and_es_check(gpu, miters):
    p, g = miters["mult12_array_wallace_flip1108"]
    r = es.run_exhaustive(p, engine="jit", devices="all")
    _check(r, g, "all")
    assert r.stats["n_devices"] == es.device_count() >= 1


def test_bad_device_list_fails_loudly(gpu, miters):
    from paper_2512_06627_b200 import _native as N
    p, _ = miters["adder8_ripple_lookahead"]
    with pytest.raises(N.NativeError, match="out of range"):
        es.run_exhaustive(p, engine="jit", devices=[0, 64])


def test_multi_device_budget_and_cancel(gpu, miters):
    p, _ = miters["mult16_array_booth"]
    r = es.run_exhaustive(p, engine="jit", cofactor="none", devices=[0, 0], budget=0.002, slice_ms=0.5)
    assert r.verdict in (es.BUDGET_EXCEEDED, es.EXHAUSTED_ZERO)
    if r.verdict == es.BUDGET_EXCEEDED:
        assert 0 < r.patterns_evaluated < 1 << 32
    r = es.run_exhaustive(p, engine="jit", devices=[0, 0], cancel=lambda: True)
    assert r.verdict == es.BUDGET_EXCEEDED and r.patterns_evaluated == 0
