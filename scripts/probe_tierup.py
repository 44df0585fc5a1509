"""Dev probe: the auto policy's tier-up on a re-run program (mult16): depth,
ptxas level, JIT and device time per call."""
import sys, time
sys.path.insert(0, '.')
import bench
from paper_2512_06627_b200 import es, shard
shard.alu_peak(0)
x, _ = bench.build_workload("mult16")
sm = bench._Sub(x)
for i in range(40):
    t = time.perf_counter()
    r = es.es_check(sm)
    w = 1e3 * (time.perf_counter() - t)
    s = r.stats
    if i < 6 or i % 8 == 7:
        print(f"call {i}: k={s.get('cofactor_pis')} O{s.get('jit_opt')} jit={s.get('jit_ms'):.0f}ms "
              f"dev={s.get('device_ms'):.2f}ms wall={w:.1f}ms", flush=True)
