"""Random simulation (K3, es_sim.cu) on the GPU: node-value matrices, PE
classes and counterexample refinement bit-exact with the reference (golden
fixtures from tests/golden/make_golden_sim.py) and with the numpy oracle on
larger drives."""
import json
import os
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200 import sim
from paper_2512_06627_b200.xag import XagBuilder, random_xag
from tests.golden import recipes
from tests.test_sim import GOLD, cls_sha, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rows():
    return json.load(open(GOLD))["rows"]


def test_simulate_golden(rows, gpu):
    for r in rows:
        x = recipes.build_sim(r)
        vals = sim.simulate(x, sim.random_pi_words(x.num_pis, r["words"], r["sim_seed"]))
        assert sha(vals.tobytes()) == r["vals_sha"], r
        assert round(float(sim.ones_fraction(vals).sum()), 9) == r["ones_sum"]


def test_ones_and_features_golden(rows, gpu):
    """es_sim_ones (popcount on the device) and stability_entropy vs the
    reference's features.py:165-180 sums; per-node equality with the oracle."""
    for r in rows:
        x = recipes.build_sim(r)
        pw = sim.random_pi_words(x.num_pis, r["words"], r["sim_seed"])
        cnt = sim.ones_counts(x, pw)
        assert cnt.dtype == np.int64 and sha(cnt.tobytes()) == r["ones_counts_sha"], r
        stab, ent = sim.stability_entropy(x, r["words"], r["sim_seed"])
        assert round(sum(stab), 9) == r["stability_sum"], r
        assert round(sum(ent), 9) == r["entropy_sum"], r
        if r["words"] <= 64:
            ostab, oent = O.stability_entropy(x, pw)
            assert stab == ostab and ent == oent


def test_classes_golden(rows, gpu):
    for r in rows:
        x = recipes.build_sim(r)
        fused = sim.pe_classes(x, r["words"], r["sim_seed"])
        assert cls_sha([c.members for c in fused]) == r["classes_sha"], r
        assert all(c.representative == c.members[0][0] for c in fused)
        host = sim.build_pe_classes(sim.random_simulate(x, r["words"], r["sim_seed"]))
        assert cls_sha([c.members for c in host]) == r["classes_sha"], r
        refined = sim.refine_with_cex(x, fused, tuple(r["cex_pattern"]))
        assert cls_sha([c.members for c in refined]) == r["refined_sha"], r


def test_simulate_wide_drives_vs_oracle(gpu):
    rng = random.Random(3)
    for k in range(6):
        x = random_xag(rng.randint(2, 30), rng.randint(50, 3000), 123 + k)
        pw = sim.random_pi_words(x.num_pis, rng.choice([129, 1000, 4097]), k)
        assert np.array_equal(sim.simulate(x, pw), O.simulate(x, pw))
    m = M.gen_multiplier_miter(16, "array", "booth")
    pw = sim.random_pi_words(m.num_pis, 2048, 9)
    want = O.simulate(m, pw)
    assert np.array_equal(sim.simulate(m, pw), want)
    got = [c.members for c in sim.pe_classes(m, pi_words=pw)]
    assert got == O.pe_classes(want)


def test_simulate_edges(gpu):
    # no gates: PI rows and the constant row only
    b = XagBuilder(3)
    x = b.finish([b.pi(2)])
    pw = sim.random_pi_words(3, 5, 1)
    assert np.array_equal(sim.simulate(x, pw), O.simulate(x, pw))
    assert [c.members for c in sim.pe_classes(x, pi_words=pw)] == O.pe_classes(O.simulate(x, pw))
    # identical and complementary nodes, a dead gate
    b = XagBuilder(4)
    p = [b.pi(i) for i in range(1, 5)]
    g1 = b.add_and(p[0], p[1])
    b.add_xor(p[2], p[3])                     # dead
    g2 = b.add_or(~p[0], ~p[1])               # == ~g1
    x = b.finish([b.add_xor(g1, g2)])
    pw = sim.random_pi_words(4, 64, 2)
    vals = sim.simulate(x, pw)
    assert np.array_equal(vals, O.simulate(x, pw))
    assert [c.members for c in sim.pe_classes(x, pi_words=pw)] == O.pe_classes(vals)


def test_device_resident(gpu):
    import torch
    m = M.gen_multiplier_miter(8, "array", "booth")
    pw = sim.random_pi_words(m.num_pis, 4096, 5)
    d_pi = torch.from_numpy(pw.view(np.int64)).cuda()
    nn = 1 + m.num_pis + len(m.gates)
    d_out = torch.empty((nn, 4096), dtype=torch.int64, device="cuda")
    ds = sim.DeviceSim(m)
    for _ in range(2):
        ds.run(d_pi.data_ptr(), 4096, d_out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy().view(np.uint64), O.simulate(m, pw))
    ds.close()


def test_large_drives(gpu):
    """Drives of >= 16,384 words (one lane per word, L2-sized word tiles):
    node matrices, classes and the device-resident path equal the numpy
    oracle's, including odd word counts (a partial last CTA)."""
    import torch
    rng = random.Random(11)
    for k in range(3):
        x = random_xag(rng.randint(6, 30), rng.randint(200, 2500), 500 + k)
        pw = sim.random_pi_words(x.num_pis, rng.choice([16384, 16411, 20000]), k)
        assert np.array_equal(sim.simulate(x, pw), O.simulate(x, pw))
    m = M.gen_multiplier_miter(16, "array", "booth")
    pw = sim.random_pi_words(m.num_pis, 16389, 4)
    want = O.simulate(m, pw)
    assert np.array_equal(sim.simulate(m, pw), want)
    assert [c.members for c in sim.pe_classes(m, pi_words=pw)] == O.pe_classes(want)
    nn = 1 + m.num_pis + len(m.gates)
    d_pi = torch.from_numpy(pw.view(np.int64)).cuda()
    d_out = torch.empty((nn, pw.shape[1]), dtype=torch.int64, device="cuda")
    ds = sim.DeviceSim(m)
    ds.run(d_pi.data_ptr(), pw.shape[1], d_out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy().view(np.uint64), want)
    ds.close()


@pytest.mark.parametrize("pipe", ["0", "1"])
def test_batch_schedules_and_lanes(gpu, monkeypatch, pipe):
    """Both batch schedules (level batches; the distance-2 list schedule of
    the software-pipelined kernel, ES_SIM_PIPE) at every lanes-per-word count
    (ES_SIM_G) equal the numpy oracle, on random XAGs (ragged last batches,
    duplicate fanins, narrow tails) and the configs[2] miter."""
    monkeypatch.setenv("ES_SIM_PIPE", pipe)
    rng = random.Random(29)
    cases = [random_xag(rng.randint(2, 24), rng.randint(1, 1500), 900 + k) for k in range(4)]
    cases.append(M.gen_multiplier_miter(16, "array", "booth"))
    for g in ("1", "2", "4", "8"):
        monkeypatch.setenv("ES_SIM_G", g)
        for k, x in enumerate(cases):
            pw = sim.random_pi_words(x.num_pis, rng.choice([1, 33, 300, 2051]), k)
            assert np.array_equal(sim.simulate(x, pw), O.simulate(x, pw)), (pipe, g, k)
