"""Dev probe: K1 (mult16) at a cofactor depth / CTA size under the register
cap in ES_MAXNREG (set per process: the JIT cache is keyed by PTX)."""
import os, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import es, miter as M
k, bt = int(sys.argv[1]), int(sys.argv[2])
m = M.gen_multiplier_miter(16, "array", "booth")
p = es.compile_program(m)
ts = []
for rep in range(6):
    r = es.run_exhaustive(p, engine="jit", cofactor=k if k else "none", block_threads=bt)
    ts.append(r.stats["device_ms"])
print(f"k={k} bt={bt} cap={os.environ.get('ES_MAXNREG', '-')} {r.verdict} dev={min(ts[1:]):.3f}ms "
      f"regs={r.stats['regs_per_thread']} jit={r.stats['jit_ms']:.0f}", flush=True)
