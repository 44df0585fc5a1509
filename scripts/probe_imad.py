"""Dev probe: K1 on mult16 with the FMA-pipe-aware LUT mapping
(ES_IMAD_COST = area weight of a 2-input LUT over a word-uniform node,
which emit_body_ptx turns into an IMAD).  One process per cost value:
    ES_IMAD_COST=0.4 python scripts/probe_imad.py 4 5
"""
import os, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M, es

m = M.gen_multiplier_miter(16, "array", "booth")
p = es.compile_program(m)
G = p.num_gates
c = os.environ.get("ES_IMAD_COST", "1.0")
for k in [int(a) for a in sys.argv[1:]] or [4]:
    pipes = es.map_pipes(p, k)
    ts = []
    for rep in range(8):
        r = es.run_exhaustive(p, engine="jit", cofactor=k, jit_parts=1)
        assert r.verdict == es.EXHAUSTED_ZERO, r
        ts.append(r.stats['device_ms'])
    t = min(ts[1:])
    print(f"cost={c} k={k} dev={t:.4f}ms med={sorted(ts[1:])[3]:.4f} rate={G * 2**32 / (t * 1e-3):.3e} "
          f"lop3={pipes['lop3']} imad={pipes['imad']} regs={r.stats.get('regs_per_thread')} "
          f"jit={r.stats.get('jit_ms'):.0f}ms", flush=True)
