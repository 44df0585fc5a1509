"""Dev probe: mult16 with PI `pi` fixed to 0 and to 1 (two 31-PI programs),
each swept with k cofactor PIs in throughput mode -- the cost of a k+1
variant evaluated as two half-bodies (loop fission)."""
import sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import es, miter as M
from paper_2512_06627_b200.xag import XagBuilder, FALSE, TRUE, GateKind


def fix(x, fixes):
    b = XagBuilder(x.num_pis - len(fixes))
    lits = [FALSE]
    j = 0
    for i in range(1, x.num_pis + 1):
        if i in fixes:
            lits.append(TRUE if fixes[i] else FALSE)
        else:
            j += 1
            lits.append(b.pi(j))
    for g in x.gates:
        a = lits[g.in0.node]; a = ~a if g.in0.neg else a
        c = lits[g.in1.node]; c = ~c if g.in1.neg else c
        lits.append(b.add_xor(a, c) if g.kind == GateKind.XOR else b.add_and(a, c))
    o = x.outputs[0]
    r = lits[o.node]
    return b.finish([~r if o.neg else r])


m = M.gen_multiplier_miter(16, "array", "booth")
pi = int(sys.argv[1]) if len(sys.argv) > 1 else 28
tot = 0.0
for v in (0, 1):
    p = es.compile_program(fix(m, {pi: v}))
    ts = [es.run_exhaustive(p, engine="jit", cofactor=int(sys.argv[2]) if len(sys.argv) > 2 else "throughput").stats for _ in range(6)]
    t = min(s["device_ms"] for s in ts[1:])
    tot += t
    print(f"PI{pi}={v}: {t:.4f} ms k={ts[-1]['cofactor_pis']} luts={ts[-1]['luts']} regs={ts[-1]['regs_per_thread']}",
          flush=True)
print(f"sum {tot:.4f} ms (one 32-PI sweep)")
