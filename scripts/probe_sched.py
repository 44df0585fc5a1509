"""Dev probe: K1 device time on mult16 for forced cofactor depths under the
schedule knobs in the environment (ES_LIST_SCHED window)."""
import os, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M, es

m = M.gen_multiplier_miter(16, "array", "booth")
p = es.compile_program(m)
G = p.num_gates
for k in [int(a) for a in sys.argv[1:]] or [3, 4]:
    st = es.map_stats(p, k)
    ts = []
    for rep in range(8):
        r = es.run_exhaustive(p, engine="jit", cofactor=k)
        ts.append(r.stats['device_ms'])
    t = min(ts[2:])
    print(f"LIST={os.environ.get('ES_LIST_SCHED', '-')} k={k} dev={t:.3f}ms rate={G * 2**32 / (t * 1e-3):.3e} "
          f"luts={st['luts']} live={st['peak_live']} regs={r.stats.get('regs_per_thread')}", flush=True)
