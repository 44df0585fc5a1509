"""Miter construction and the benchmark-circuit generators for the ES configs.

``build_miter``/``or_reduce``/``copy_into`` and the "array"/"diagonal"
multipliers reproduce the reference constructions (cecprove/miter.py:27-134)
gate for gate, so their miters are identical to the reference's.  The
generators the reference lacks and BASELINE.json's configs need are new:
carry-lookahead adder (config 1), Wallace-tree multiplier (config 2) and
unsigned radix-4 Booth multiplier (config 3).  Operand convention as the
reference (miter.py:122-134): PIs 1..w are operand A LSB first, w+1..2w
operand B; outputs LSB first.
"""

from __future__ import annotations

import random

from .xag import FALSE, TRUE, Gate, GateKind, Lit, Xag, XagBuilder


class InterfaceMismatch(ValueError):
    pass


class WidthOutOfRange(ValueError):
    pass


def copy_into(b: XagBuilder, xag, pi_lits: list[Lit] | None = None) -> list[Lit]:
    """Replay a circuit into a builder; returns its mapped outputs."""
    lit_of: list[Lit] = [FALSE]
    lit_of.extend(pi_lits if pi_lits is not None
                  else [b.pi(i) for i in range(1, xag.num_pis + 1)])

    def m(l: Lit) -> Lit:
        base = lit_of[l.node]
        return Lit(base.node, base.neg != l.neg)

    for g in xag.gates:
        x, y = m(g.in0), m(g.in1)
        lit_of.append(b.add_and(x, y) if g.kind == GateKind.AND else b.add_xor(x, y))
    return [m(o) for o in xag.outputs]


def or_reduce(b: XagBuilder, lits: list[Lit]) -> Lit:
    """Balanced pairwise OR tree, left to right; empty -> FALSE."""
    if not lits:
        return FALSE
    while len(lits) > 1:
        nxt = []
        for k in range(0, len(lits), 2):
            nxt.append(b.add_or(lits[k], lits[k + 1]) if k + 1 < len(lits) else lits[k])
        lits = nxt
    return lits[0]


def build_miter(a, c) -> Xag:
    """XOR corresponding outputs and OR-reduce them (miter.py:52-62)."""
    if a.num_pis != c.num_pis:
        raise InterfaceMismatch(f"PI counts differ: {a.num_pis} vs {c.num_pis}")
    if len(a.outputs) != len(c.outputs):
        raise InterfaceMismatch(
            f"output counts differ: {len(a.outputs)} vs {len(c.outputs)}")
    b = XagBuilder(a.num_pis)
    oa = copy_into(b, a)
    oc = copy_into(b, c)
    return b.finish([or_reduce(b, [b.add_xor(x, y) for x, y in zip(oa, oc)])])


# --- adders -----------------------------------------------------------------

def full_add(b: XagBuilder, x: Lit, y: Lit, cin: Lit) -> tuple[Lit, Lit]:
    """Sum and carry with the reference's gate structure (miter.py:65-69)."""
    t = b.add_xor(x, y)
    s = b.add_xor(t, cin)
    return s, b.add_or(b.add_and(x, y), b.add_and(t, cin))


def half_add(b: XagBuilder, x: Lit, y: Lit) -> tuple[Lit, Lit]:
    return b.add_xor(x, y), b.add_and(x, y)


def ripple_add(b: XagBuilder, xs: list[Lit], ys: list[Lit]) -> list[Lit]:
    """Ripple-carry sum, width+1 bits (miter.py:72-81)."""
    w = max(len(xs), len(ys))
    xs = xs + [FALSE] * (w - len(xs))
    ys = ys + [FALSE] * (w - len(ys))
    out, carry = [], FALSE
    for x, y in zip(xs, ys):
        s, carry = full_add(b, x, y, carry)
        out.append(s)
    out.append(carry)
    return out


def lookahead_add(b: XagBuilder, xs: list[Lit], ys: list[Lit],
                  block: int = 4) -> list[Lit]:
    """Two-level carry-lookahead sum, width+1 bits.

    Bit generate g=x&y and propagate p=x^y; inside each block every carry is
    the flattened sum-of-products c[i+1] = g[i] | p[i]g[i-1] | ... |
    p[i]..p[lo]c[lo]; block generate/propagate feed a second lookahead level
    that produces the block carry-ins directly from c0 = 0.
    """
    w = len(xs)
    assert len(ys) == w
    g = [b.add_and(x, y) for x, y in zip(xs, ys)]
    p = [b.add_xor(x, y) for x, y in zip(xs, ys)]
    blocks = [(lo, min(lo + block, w)) for lo in range(0, w, block)]

    def span_gp(lo: int, hi: int) -> tuple[Lit, Lit]:
        terms = []
        for i in range(lo, hi):
            t = g[i]
            for k in range(i + 1, hi):
                t = b.add_and(t, p[k])
            terms.append(t)
        prop = TRUE
        for k in range(lo, hi):
            prop = b.add_and(prop, p[k])
        return or_reduce(b, terms), prop

    bgp = [span_gp(lo, hi) for lo, hi in blocks]
    cin = [FALSE]
    for j in range(1, len(blocks) + 1):
        terms = []
        for i in range(j):
            t = bgp[i][0]
            for k in range(i + 1, j):
                t = b.add_and(t, bgp[k][1])
            terms.append(t)
        cin.append(or_reduce(b, terms))
    out: list[Lit] = []
    for (lo, hi), c0 in zip(blocks, cin):
        for i in range(lo, hi):
            terms = []
            for j in range(lo, i):
                t = g[j]
                for k in range(j + 1, i):
                    t = b.add_and(t, p[k])
                terms.append(t)
            t = c0
            for k in range(lo, i):
                t = b.add_and(t, p[k])
            terms.append(t)
            out.append(b.add_xor(p[i], or_reduce(b, terms)))
    out.append(cin[-1])
    return out


def gen_adder(width: int, arch: str) -> Xag:
    """Unsigned width-bit adder, width+1 outputs; arch 'ripple' or 'lookahead'."""
    if not 1 <= width <= 64:
        raise WidthOutOfRange(f"width {width} outside [1, 64]")
    b = XagBuilder(2 * width)
    xs = [b.pi(i) for i in range(1, width + 1)]
    ys = [b.pi(i) for i in range(width + 1, 2 * width + 1)]
    if arch == "ripple":
        outs = ripple_add(b, xs, ys)
    elif arch == "lookahead":
        outs = lookahead_add(b, xs, ys)
    else:
        raise ValueError(f"unknown adder architecture {arch!r}")
    return b.finish(outs)


# --- multipliers ------------------------------------------------------------

def _mult_array(b: XagBuilder, aa: list[Lit], bb: list[Lit]) -> list[Lit]:
    """Row-by-row accumulation through ripple adders (miter.py:84-90)."""
    n = len(aa)
    acc = [b.add_and(aa[j], bb[0]) for j in range(n)]
    for i in range(1, n):
        acc = ripple_add(b, acc, [FALSE] * i + [b.add_and(aa[j], bb[i]) for j in range(n)])
    return acc[: 2 * n]


def _mult_diagonal(b: XagBuilder, aa: list[Lit], bb: list[Lit]) -> list[Lit]:
    """Carry-save rows, carries shifted one column, final ripple (miter.py:93-116)."""
    n = len(aa)
    w = 2 * n
    sums = [FALSE] * w
    carries = [FALSE] * w
    for i in range(n):
        row = [FALSE] * w
        for j in range(n):
            row[i + j] = b.add_and(aa[j], bb[i])
        ns, nc = [FALSE] * w, [FALSE] * w
        for k in range(w):
            s, c = full_add(b, sums[k], carries[k], row[k])
            ns[k] = s
            if k + 1 < w:
                nc[k + 1] = c
        sums, carries = ns, nc
    return ripple_add(b, sums, carries)[:w]


def _compress_columns(b: XagBuilder, cols: list[list[Lit]]) -> list[Lit]:
    """Wallace reduction of bit columns, then a ripple-carry final add.

    Each layer turns every full triple of a column into a full adder and a
    leftover pair into a half adder (Wallace's greedy rule), until no column
    is taller than two; the two remaining rows go through ripple_add.
    """
    w = len(cols)
    cols = [[l for l in c if l != FALSE] for c in cols]
    while max((len(c) for c in cols), default=0) > 2:
        nxt: list[list[Lit]] = [[] for _ in range(w)]
        for k, col in enumerate(cols):
            i = 0
            while len(col) - i >= 3:
                s, c = full_add(b, col[i], col[i + 1], col[i + 2])
                nxt[k].append(s)
                if k + 1 < w:
                    nxt[k + 1].append(c)
                i += 3
            if len(col) - i == 2:
                s, c = half_add(b, col[i], col[i + 1])
                nxt[k].append(s)
                if k + 1 < w:
                    nxt[k + 1].append(c)
            elif len(col) - i == 1:
                nxt[k].append(col[i])
        cols = [[l for l in c if l != FALSE] for c in nxt]
    row0 = [c[0] if len(c) > 0 else FALSE for c in cols]
    row1 = [c[1] if len(c) > 1 else FALSE for c in cols]
    return ripple_add(b, row0, row1)[:w]


def _mult_wallace(b: XagBuilder, aa: list[Lit], bb: list[Lit]) -> list[Lit]:
    n = len(aa)
    cols: list[list[Lit]] = [[] for _ in range(2 * n)]
    for i in range(n):
        for j in range(n):
            cols[i + j].append(b.add_and(aa[j], bb[i]))
    return _compress_columns(b, cols)


def _mult_booth4(b: XagBuilder, aa: list[Lit], bb: list[Lit]) -> list[Lit]:
    """Unsigned radix-4 (modified) Booth with Wallace reduction.

    B is zero-extended so its recoding digits d_i = -2b[2i+1] + b[2i] +
    b[2i-1] in {-2..2} (b[-1] = 0), i = 0..n/2, give B = sum d_i 4^i.
    Row i is |d_i|*A selected per bit (one: A, two: A<<1) and inverted when
    d_i < 0, plus the +1 of the two's-complement negation at column 2i.  Sign
    extension uses the constant-compensation identity
        -s 2^(n+1) = (~s) 2^(n+1) - 2^(n+1),
    so each row contributes ~s_i at column 2i+n+1 and the constant
    -sum_i 2^(2i+n+1) mod 2^(2n) is folded in as TRUE bits.
    """
    n = len(aa)
    w = 2 * n
    bits = [FALSE] + bb + [FALSE, FALSE]  # bits[k+1] = b[k], b[-1] = 0

    def bit(k: int) -> Lit:
        return bits[k + 1]

    cols: list[list[Lit]] = [[] for _ in range(w)]
    const = 0
    for i in range(n // 2 + 1):
        hi, mid, lo = bit(2 * i + 1), bit(2 * i), bit(2 * i - 1)
        one = b.add_xor(mid, lo)
        two = b.add_or(b.add_and(hi, b.add_and(~mid, ~lo)),
                       b.add_and(~hi, b.add_and(mid, lo)))
        neg = b.add_and(hi, ~b.add_and(mid, lo))
        for j in range(n + 1):
            aj = aa[j] if j < n else FALSE
            aj1 = aa[j - 1] if j >= 1 else FALSE
            pp = b.add_xor(b.add_or(b.add_and(one, aj), b.add_and(two, aj1)), neg)
            col = 2 * i + j
            if col < w:
                cols[col].append(pp)
        if 2 * i < w:
            cols[2 * i].append(neg)
        if 2 * i + n + 1 < w:
            cols[2 * i + n + 1].append(~neg)
        const -= 1 << (2 * i + n + 1)
    const %= 1 << w
    for k in range(w):
        if (const >> k) & 1:
            cols[k].append(TRUE)
    # fold constant TRUE bits pairwise before the tree so no column holds
    # constants the builder cannot absorb
    for k in range(w):
        ones = sum(1 for l in cols[k] if l == TRUE)
        cols[k] = [l for l in cols[k] if l != TRUE and l != FALSE]
        carry_ones, rem = divmod(ones, 2)
        if rem:
            cols[k].append(TRUE)
        if carry_ones and k + 1 < w:
            cols[k + 1].extend([TRUE] * carry_ones)
    return _compress_columns(b, cols)


_MULTS = {"array": _mult_array, "diagonal": _mult_diagonal,
          "wallace": _mult_wallace, "booth": _mult_booth4}


def gen_multiplier(width: int, arch: str) -> Xag:
    """Unsigned width x width multiplier, 2*width outputs, LSB first."""
    if not 2 <= width <= 32:
        raise WidthOutOfRange(f"width {width} outside [2, 32]")
    if arch not in _MULTS:
        raise ValueError(f"unknown architecture {arch!r}")
    if arch == "booth" and width % 2:
        raise WidthOutOfRange("radix-4 Booth generator needs an even width")
    b = XagBuilder(2 * width)
    aa = [b.pi(i) for i in range(1, width + 1)]
    bb = [b.pi(i) for i in range(width + 1, 2 * width + 1)]
    return b.finish(_MULTS[arch](b, aa, bb))


def gen_multiplier_miter(width: int, arch_a: str, arch_b: str) -> Xag:
    return build_miter(gen_multiplier(width, arch_a), gen_multiplier(width, arch_b))


def gen_adder_miter(width: int, arch_a: str = "ripple",
                    arch_b: str = "lookahead") -> Xag:
    return build_miter(gen_adder(width, arch_a), gen_adder(width, arch_b))


def flip_gate(xag: Xag, idx: int) -> Xag:
    """Single-gate fault: gate idx AND<->XOR (the reference's fault model)."""
    g = xag.gates[idx]
    k = GateKind.XOR if g.kind == GateKind.AND else GateKind.AND
    return Xag(xag.num_pis, xag.gates[:idx] + (Gate(k, g.in0, g.in1),) + xag.gates[idx + 1:],
               xag.outputs)


def mutate(xag: Xag, seed: int, check_pis: int = 16) -> Xag:
    """Flip one gate AND<->XOR, verified to change the function at <= check_pis PIs.

    Same draw sequence as the reference (miter.py:141-162).  Verification
    uses this package's truth table (exhaustive, small widths only).
    """
    if not xag.gates:
        raise ValueError("no gates to mutate")
    rng = random.Random(seed)
    verify = xag.num_pis <= check_pis and len(xag.outputs) == 1
    before = truth_table(xag) if verify else None
    for _ in range(10 * len(xag.gates)):
        idx = rng.randrange(len(xag.gates))
        mutant = flip_gate(xag, idx)
        if not verify or truth_table(mutant) != before:
            return mutant
    raise ValueError("could not find a function-changing mutation")


# --- scalar evaluation (witness re-check, small truth tables) ---------------

def evaluate(xag, bits) -> int:
    """Single output on one assignment, bit i -> PI i+1 (the witness re-check
    es_check performs, es.py:360-361)."""
    vals = [0] * (1 + xag.num_pis + len(xag.gates))
    if len(bits) != xag.num_pis:
        raise ValueError(f"expected {xag.num_pis} input bits, got {len(bits)}")
    for i, v in enumerate(bits):
        vals[1 + i] = 1 if v else 0
    base = 1 + xag.num_pis
    for i, g in enumerate(xag.gates):
        a = vals[g.in0.node] ^ int(g.in0.neg)
        c = vals[g.in1.node] ^ int(g.in1.neg)
        vals[base + i] = (a & c) if g.kind == GateKind.AND else (a ^ c)
    o = xag.outputs[0]
    return vals[o.node] ^ int(o.neg)


def truth_table(xag, max_pis: int = 22) -> int:
    """Output over all 2^n rows as one big int, bit p = row p (row p gives
    PI j the value bit j-1 of p).  Small widths only; used by ``mutate``."""
    n = xag.num_pis
    if n > max_pis:
        raise ValueError(f"truth table over {n} PIs exceeds cap {max_pis}")
    total = 1 << n
    mask = (1 << total) - 1
    vals = [0] * (1 + n + len(xag.gates))
    for j in range(n):
        period = 1 << (j + 1)
        block = ((1 << (1 << j)) - 1) << (1 << j)
        vals[1 + j] = block * (mask // ((1 << period) - 1)) if total > period else block
    base = 1 + n
    for i, g in enumerate(xag.gates):
        a = vals[g.in0.node] ^ (mask if g.in0.neg else 0)
        c = vals[g.in1.node] ^ (mask if g.in1.neg else 0)
        vals[base + i] = (a & c) if g.kind == GateKind.AND else (a ^ c)
    o = xag.outputs[0]
    return vals[o.node] ^ (mask if o.neg else 0)
