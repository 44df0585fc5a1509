"""Dev probe: K1 on top-PI cofactor expansions of mult16 (OR of the 2^k
cofactors as an (n-k)-PI XAG).  Times the reduced sweep, reports the
original-metric rate G*2^n/t."""
import itertools, sys, time
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M, es
from paper_2512_06627_b200.xag import XagBuilder, FALSE, TRUE, GateKind


def cofactor_expand(x, k):
    n = x.num_pis - k
    b = XagBuilder(n)
    outs = []
    for assign in itertools.product([0, 1], repeat=k):
        lits = [FALSE] + [b.pi(i) for i in range(1, n + 1)] + [TRUE if v else FALSE for v in assign]
        for g in x.gates:
            a = lits[g.in0.node]; a = ~a if g.in0.neg else a
            c = lits[g.in1.node]; c = ~c if g.in1.neg else c
            lits.append(b.add_xor(a, c) if g.kind == GateKind.XOR else b.add_and(a, c))
        o = x.outputs[0]; r = lits[o.node]; outs.append(~r if o.neg else r)
    return b.finish([M.or_reduce(b, outs)])


BTS = (256, 512)
m = M.gen_multiplier_miter(16, "array", "booth")
G = es.compile_program(m).num_gates
for k in [int(a) for a in sys.argv[1:]] or [0, 1, 2, 3]:
    y = cofactor_expand(m, k) if k else m
    p = es.compile_program(y)
    for bt in BTS:
        ts = []
        for rep in range(6):
            r = es.run_exhaustive(p, engine="jit", block_threads=bt)
            ts.append(r.stats['device_ms'])
        t = min(ts[1:])
        print(f"k={k} bt={bt} {r.verdict} dev={t:.3f}ms rate={G * 2**32 / (t * 1e-3):.3e} "
              f"luts={r.stats.get('luts')} regs={r.stats.get('regs_per_thread')} jit={r.stats.get('jit_ms'):.0f}ms",
              flush=True)
