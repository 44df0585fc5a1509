"""Dev probe: host overhead of a warm es_check on mult16 (throughput mode):
Python compile_program, native es_run wall time vs device time."""
import sys, time
sys.path.insert(0, '.')
from paper_2512_06627_b200 import es, miter as M
from paper_2512_06627_b200.verdict import CheckResult

class _Sub:
    def __init__(self, x): self.circuit = x

x = M.gen_multiplier_miter(16, "array", "booth")
sm = _Sub(x)
for _ in range(5):
    es.es_check(sm, engine="jit", cofactor="throughput")
rows = []
for _ in range(30):
    t0 = time.perf_counter()
    p = es.compile_program(x)
    t1 = time.perf_counter()
    r = es.run_exhaustive(p, engine="jit", cofactor="throughput")
    t2 = time.perf_counter()
    rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, r.stats["engine_wall_ms"], r.stats["device_ms"]))
rows.sort(key=lambda r: r[1])
m = rows[len(rows) // 2]
print(f"compile {m[0]:.3f} ms  run_exhaustive {m[1]:.3f} ms  native wall {m[2]:.3f} ms  device {m[3]:.3f} ms")
t = time.perf_counter()
for _ in range(30):
    es.es_check(sm, engine="jit", cofactor="throughput")
print(f"es_check {(time.perf_counter() - t) / 30 * 1e3:.3f} ms per call")
