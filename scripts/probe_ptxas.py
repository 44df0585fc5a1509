"""Dev probe: JIT (PTX -> SASS) time vs kernel time on mult16 per cofactor
depth under ES_PTXAS_O (run with ES_JIT_CACHE=0)."""
import os, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M, es

m = M.gen_multiplier_miter(16, "array", "booth")
p = es.compile_program(m)
for k in [int(a) for a in sys.argv[1:]] or [0, 2, 4]:
    r = es.run_exhaustive(p, engine="jit", cofactor=k)
    jit = r.stats.get("jit_ms")
    ts = [es.run_exhaustive(p, engine="jit", cofactor=k).stats["device_ms"] for _ in range(4)]
    print(f"O={os.environ.get('ES_PTXAS_O', '3')} k={k} jit={jit:.0f}ms dev={min(ts):.3f}ms "
          f"regs={r.stats.get('regs_per_thread')}", flush=True)
