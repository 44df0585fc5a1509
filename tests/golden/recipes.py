"""Deterministic recipes for every golden circuit (shared by the fixture
generator and the tests that replay the fixtures).

A recipe is a small dict; ``build_*`` turns it into an ``Xag`` with this
repo's generators.  ``xag_sha``/``prog_sha`` fingerprint circuits and
instruction programs so fixtures stay small while still pinning
gate-for-gate and instruction-for-instruction parity.
"""

from __future__ import annotations

import hashlib
import json
import random

from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.xag import random_xag


def xag_sha(x) -> str:
    body = [x.num_pis,
            [[int(g.kind), g.in0.node * 2 + int(g.in0.neg), g.in1.node * 2 + int(g.in1.neg)]
             for g in x.gates],
            [o.node * 2 + int(o.neg) for o in x.outputs]]
    return hashlib.sha256(json.dumps(body, separators=(",", ":")).encode()).hexdigest()[:20]


def prog_sha(rows, num_registers: int) -> str:
    body = [num_registers, [[int(v) for v in r] for r in rows]]
    return hashlib.sha256(json.dumps(body, separators=(",", ":")).encode()).hexdigest()[:20]


# --- random populations -------------------------------------------------------

def random_population() -> list[dict]:
    specs = []
    # test_acceptance.py:82-101 oracle-agreement population
    rng = random.Random(2024)
    for k in range(500):
        specs.append({"pop": "acceptance500", "n_pis": rng.randint(1, 14),
                      "n_gates": rng.randint(0, 300), "seed": k})
    # test_es.py:58-67 and :70-78 hypothesis ranges
    for s in range(0, 301):
        specs.append({"pop": "tt6x40", "n_pis": 6, "n_gates": 40, "seed": s})
    for s in range(0, 101):
        specs.append({"pop": "workers7x50", "n_pis": 7, "n_gates": 50, "seed": s})
    # wider random cones: multi-word / multi-batch geometry on the GPU
    rng = random.Random(7)
    for k in range(60):
        specs.append({"pop": "wide", "n_pis": rng.randint(15, 24),
                      "n_gates": rng.randint(100, 1500), "seed": 10_000 + k})
    return specs


def build_random(spec: dict):
    return random_xag(spec["n_pis"], spec["n_gates"], spec["seed"])


# --- named miters -------------------------------------------------------------

# single-gate faults of the config miters whose reference min-index witness
# is deep (found by tests/golden/find_deep_faults.py; the index itself is the
# fixture the reference run pins)
DEEP_FAULTS = {
    "mult12_array_wallace": [1108, 1210, 941],
    "mult16_array_booth": [2204, 1953, 1406, 1882, 1220],
}


def miter_population() -> list[dict]:
    specs: list[dict] = []
    for w in range(2, 15):
        specs.append({"name": f"mult{w}_array_diagonal", "kind": "mult", "w": w,
                      "a": "array", "b": "diagonal", "full_program": w == 3})
    for w in range(1, 9):
        specs.append({"name": f"adder{w}_ripple_lookahead", "kind": "adder", "w": w,
                      "a": "ripple", "b": "lookahead", "full_program": w == 8})
    for w in range(3, 13):
        specs.append({"name": f"mult{w}_array_wallace", "kind": "mult", "w": w,
                      "a": "array", "b": "wallace"})
    for w in range(2, 15, 2):
        specs.append({"name": f"mult{w}_array_booth", "kind": "mult", "w": w,
                      "a": "array", "b": "booth"})
    # the reference's own fault model on its own miters (mutate, miter.py:141)
    for w in range(3, 9):
        for s in range(6):
            specs.append({"name": f"mult{w}_array_diagonal_mut{s}", "kind": "mult", "w": w,
                          "a": "array", "b": "diagonal", "mutate_seed": s})
    for w in (4, 6, 8):
        for s in range(4):
            specs.append({"name": f"adder{w}_ripple_lookahead_mut{s}", "kind": "adder",
                          "w": w, "a": "ripple", "b": "lookahead", "mutate_seed": s})
    for s in range(4):
        specs.append({"name": f"mult8_array_booth_mut{s}", "kind": "mult", "w": 8,
                      "a": "array", "b": "booth", "mutate_seed": s})
    for base, idxs in DEEP_FAULTS.items():
        w = int(base[4:6])
        _, a, b = base.split("_")
        for gi in idxs:
            specs.append({"name": f"{base}_flip{gi}", "kind": "mult", "w": w, "a": a, "b": b,
                          "flip_gate": gi})
    specs.append({"name": "mult16_array_booth", "kind": "mult", "w": 16, "a": "array",
                  "b": "booth", "ref_workers": 8})
    return specs


def build_miter_recipe(spec: dict):
    if spec["kind"] == "mult":
        x = M.gen_multiplier_miter(spec["w"], spec["a"], spec["b"])
    elif spec["kind"] == "adder":
        x = M.gen_adder_miter(spec["w"], spec["a"], spec["b"])
    else:
        raise ValueError(spec["kind"])
    if "mutate_seed" in spec:
        x = M.mutate(x, seed=spec["mutate_seed"])
    if "flip_gate" in spec:
        x = M.flip_gate(x, spec["flip_gate"])
    return x


def build_with_reference(spec: dict, ref_miter, ref_xag):
    """Same circuit from the reference's own generators, when it has them."""
    if spec["kind"] != "mult" or {spec["a"], spec["b"]} - {"array", "diagonal"}:
        return None
    x = ref_miter.gen_multiplier_miter(spec["w"], spec["a"], spec["b"])
    if "mutate_seed" in spec:
        x = ref_miter.mutate(x, seed=spec["mutate_seed"])
    if "flip_gate" in spec:
        return None
    return x


# --- random-simulation population (make_golden_sim.py, tests/test_sim*.py) ---

def sim_population() -> list[dict]:
    """Circuits x drives: random XAGs, multiplier/adder miters, the config
    miters at the sweep's 64-word default (sweep.py:313)."""
    specs = []
    rng = random.Random(77)
    for k in range(40):
        specs.append({"kind": "random", "n_pis": rng.randint(1, 20), "n_gates": rng.randint(0, 600),
                      "seed": 7000 + k, "words": rng.choice([1, 2, 3, 17, 64, 100]), "sim_seed": k})
    for w, a, b in [(4, "array", "diagonal"), (6, "array", "diagonal"), (8, "array", "diagonal"),
                    (8, "array", "booth"), (12, "array", "wallace"), (16, "array", "booth")]:
        for words, seed in [(1, 0), (64, 0), (64, 3), (257, 1)]:
            specs.append({"kind": "mult", "width": w, "a": a, "b": b, "words": words, "sim_seed": seed})
    specs.append({"kind": "adder", "width": 8, "words": 64, "sim_seed": 0})
    return specs


def build_sim(spec):
    if spec["kind"] == "random":
        return random_xag(spec["n_pis"], spec["n_gates"], spec["seed"])
    if spec["kind"] == "mult":
        return M.gen_multiplier_miter(spec["width"], spec["a"], spec["b"])
    return M.gen_adder_miter(spec["width"])


# --- AIGER population (make_golden_aiger.py, tests/test_aiger.py) -------------

def aiger_population() -> list[dict]:
    specs = []
    rng = random.Random(91)
    for k in range(30):
        specs.append({"kind": "random", "n_pis": rng.randint(1, 16), "n_gates": rng.randint(0, 400),
                      "seed": 4000 + k, "shuffle": k % 3 == 0})
    for w, a, b in [(3, "array", "diagonal"), (4, "array", "booth"), (6, "array", "wallace"),
                    (8, "array", "booth"), (12, "array", "wallace"), (16, "array", "booth")]:
        specs.append({"kind": "mult", "width": w, "a": a, "b": b, "shuffle": w == 6})
    specs.append({"kind": "adder", "width": 8, "shuffle": True})
    return specs


def build_aiger_circuit(spec):
    return build_sim(spec)


def to_binary_aiger(ascii_bytes: bytes) -> bytes:
    """Binary AIGER of an ASCII file whose ANDs are numbered consecutively
    after the inputs with lhs > rhs0 >= rhs1 (write_aiger's form)."""
    lines = ascii_bytes.decode().strip().split("\n")
    m, i, l, o, a = (int(t) for t in lines[0].split()[1:6])
    outs = lines[1 + i:1 + i + o]
    ands = [tuple(int(t) for t in ln.split()) for ln in lines[1 + i + o:1 + i + o + a]]
    out = bytearray(f"aig {m} {i} {l} {o} {a}\n".encode())
    for ln in outs:
        out += (ln + "\n").encode()

    def varint(x):
        while True:
            byte = x & 0x7F
            x >>= 7
            if x:
                out.append(byte | 0x80)
            else:
                out.append(byte)
                return

    for lhs, r0, r1 in ands:
        varint(lhs - r0)
        varint(r0 - r1)
    return bytes(out)


def shuffled_ascii(ascii_bytes: bytes, seed: int) -> bytes:
    """Same ASCII file with the AND lines in a seeded random order (the
    reader must DFS out-of-order definitions, aiger.py:63-92)."""
    lines = ascii_bytes.decode().strip().split("\n")
    i, o, a = (int(t) for t in lines[0].split()[2:3] + lines[0].split()[4:6])
    head, body = lines[:1 + i + o], lines[1 + i + o:]
    random.Random(seed).shuffle(body)
    return ("\n".join(head + body) + "\n").encode()


AIGER_ERROR_CASES = [
    b"",
    b"aag 1 1 0 1 0",
    b"xyz 1 1 0 1 0\n2\n2\n",
    b"aag 1 1 0\n",
    b"aag a 1 0 1 0\n2\n2\n",
    b"aag 3 1 1 1 1\n2\n4 2\n6\n6 2 4\n",
    b"aag 1 2 0 1 0\n2\n4\n2\n",
    b"aag 2 1 0 1 1\n2\n4\n4 2 8\n",
    b"aag 3 1 0 1 2\n2\n4\n4 6 2\n6 4 2\n",
    b"aag 2 1 0 1 1\n2\n4\n4 2\n",
    b"aag 2 1 0 1 1\n3\n4\n4 2 2\n",
    b"aag 2 1 0 1 1\n2\n9\n4 2 2\n",
    b"aag 2 1 0 1 1 1\n2\n4\n4 2 2\n",
    b"aag 2 1 0 1 1\n2\n4\n",
    b"aig 2 1 0 1 1\n4\n",
    b"aig 2 1 0 1 1\n4\n\x05\x00",
    b"aag 2 1 0 1 1\n2\n4\n2 2 2\n",
    b"aag 2 1 0 1 1\n2\n4\n4 2 x\n",
    b"aag 3 1 0 1 1\n2\n6\n4 2 2\n",
    b"aag 1 1 0 1 0\n2\n1\n",
    b"aag 1 1 0 1 0 0 0\n2\n3\n",
]


# --- sweep population (make_golden_sweep.py, tests/test_sweep_gpu.py) ---------

def sweep_population() -> list[dict]:
    specs = []
    for w in (4, 6, 8):
        specs.append({"kind": "adder", "width": w})
    for w, a, b in [(4, "array", "diagonal"), (6, "array", "wallace"), (6, "array", "booth"),
                    (8, "array", "diagonal"), (8, "array", "booth"), (10, "array", "wallace")]:
        specs.append({"kind": "mult", "width": w, "a": a, "b": b})
        for s in range(3):
            specs.append({"kind": "mult", "width": w, "a": a, "b": b, "mutate": s})
    # deep single-gate faults the 4,096 random patterns miss: refuted by ES
    for flip in (1108, 1210, 941):
        specs.append({"kind": "mult", "width": 12, "a": "array", "b": "wallace", "flip": flip})
    specs.append({"kind": "mult", "width": 12, "a": "array", "b": "wallace"})
    # a single failing pattern (random simulation cannot see it): the final
    # ES obligation must find exactly that witness
    for w, a, b, needle in [(8, "array", "booth", 0xBEEF), (10, "array", "wallace", 0x5A5A5),
                            (12, "array", "wallace", 0xC0FFEE)]:
        specs.append({"kind": "mult", "width": w, "a": a, "b": b, "needle": needle})
    return specs


def build_sweep_circuit(spec):
    x = build_sim(spec)
    if "mutate" in spec:
        x = M.mutate(x, spec["mutate"], check_pis=0)
    if "flip" in spec:
        x = M.flip_gate(x, spec["flip"])
    if "needle" in spec:  # OR a single minterm into the output: one failing pattern
        from paper_2512_06627_b200.xag import XagBuilder
        bld = XagBuilder(x.num_pis)
        (o,) = M.copy_into(bld, x)
        t = None
        for i in range(x.num_pis):
            lit = bld.pi(i + 1) if (spec["needle"] >> i) & 1 else ~bld.pi(i + 1)
            t = lit if t is None else bld.add_and(t, lit)
        x = bld.finish([bld.add_or(o, t)])
    return x
