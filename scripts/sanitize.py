"""compute-sanitizer target: small runs of every kernel (K1 with and without
cofactor copies, K2 single and batched, K3 simulation and classes)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2512_06627_b200 import es, miter as M, sim, cones
m = M.gen_multiplier_miter(8, "array", "booth")
bad = M.flip_gate(m, 300)
for x in (m, bad):
    p = es.compile_program(x)
    for engine, cof in (("jit", "none"), ("jit", 2), ("interp", "auto")):
        r = es.run_exhaustive(p, engine=engine, cofactor=cof)
        print(engine, cof, r.verdict, r.witness_index)
b = cones.config4_batch(200)
res = b.run_arrays()
print("batch", len(res), int((res["verdict"] == 1).sum()))
pw = sim.random_pi_words(m.num_pis, 100, 0)
assert sim.simulate(m, pw).shape[1] == 100
print("classes", len(sim.pe_classes(m, pi_words=pw)))
for words in (20_000, 40_000):  # K3 at 4 and 1 lanes per word (100 words: 8)
    pw = sim.random_pi_words(m.num_pis, words, 1)
    assert sim.simulate(m, pw).shape[1] == words
print("ones", int(sim.ones_counts(m, pw).sum()))
