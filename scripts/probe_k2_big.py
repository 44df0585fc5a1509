"""Dev probe: the K2 interpreter on whole miters (mult12 / mult16 / mult16
NEQ): device time and rate per cofactor policy, for the cold-path engine
choice."""
import sys, time
sys.path.insert(0, '.')
import bench
from paper_2512_06627_b200 import es

for name in sys.argv[1:] or ["mult12", "mult16", "mult16_neq"]:
    x, _ = bench.build_workload(name)
    p = es.compile_program(x)
    for cof in ("none", "auto", "throughput"):
        ts = []
        for rep in range(3):
            t = time.perf_counter()
            r = es.run_exhaustive(p, engine="interp", cofactor=cof)
            ts.append((r.stats["device_ms"], 1e3 * (time.perf_counter() - t)))
        d, w = min(ts)
        print(f"{name} cof={cof} {r.verdict} k={r.stats.get('cofactor_pis')} dev={d:.2f}ms wall={w:.2f}ms "
              f"first_wall={ts[0][1]:.1f}ms rate={p.num_gates * 2.0 ** p.num_pis / (d * 1e-3):.3e}", flush=True)
