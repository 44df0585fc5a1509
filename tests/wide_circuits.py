"""Circuits whose live set is wider than the K2 interpreter's shared memory
(ADVICE r01, high): a butterfly network over `width` wires, every wire of
the last stage XOR-reduced.  ``eq=True`` miters the XOR chain against the
same chain in reverse order (same function, different gates), so the
output is constant 0 and the sweep must exhaust the space."""
from __future__ import annotations

import random

from paper_2512_06627_b200.xag import XagBuilder


def butterfly(n_pis: int = 24, width: int = 512, stages: int = 9, seed: int = 1, eq: bool = False):
    rng = random.Random(seed)
    b = XagBuilder(n_pis)
    pis = [b.pi(i) for i in range(1, n_pis + 1)]
    wires = []
    for i in range(width):
        x, y = rng.sample(pis, 2)
        wires.append(b.add_and(x, ~y) if i % 3 else b.add_xor(x, y))
    for s in range(stages):
        d = 1 << (s % 9)
        nw = list(wires)
        for i in range(width):
            j = i ^ d
            if i < j:
                nw[i] = b.add_xor(wires[i], wires[j])
                nw[j] = b.add_and(wires[i], ~wires[j]) if rng.random() < .5 else b.add_or(wires[i], wires[j])
        wires = nw
    acc = wires[0]
    for v in wires[1:]:
        acc = b.add_xor(acc, v)
    if not eq:
        return b.finish([acc])
    rev = wires[-1]
    for v in reversed(wires[:-1]):
        rev = b.add_xor(rev, v)
    return b.finish([b.add_xor(acc, rev)])
