"""Dev probe: K1 on mult16 at forced cofactor depths and CTA sizes (run with
ES_JIT_CACHE=0 and the knobs under test, e.g. ES_PTXAS_O=3 ES_MAXNREG=168)."""
import os, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M, es
m = M.gen_multiplier_miter(16, "array", "booth")
p = es.compile_program(m)
ks = [int(a) for a in sys.argv[1:]] or [3, 4]
for k in ks:
    for bt in (128, 256):
        ts = [es.run_exhaustive(p, engine="jit", cofactor=k, block_threads=bt).stats for _ in range(6)]
        print(f"LIST={os.environ.get('ES_LIST_SCHED', '-')} MAXNREG={os.environ.get('ES_MAXNREG', '-')} "
              f"k={k} bt={bt} dev={min(t['device_ms'] for t in ts[2:]):.3f}ms regs={ts[-1]['regs_per_thread']}",
              flush=True)
