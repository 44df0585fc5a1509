"""Dev probe: cold time-to-verdict (fresh process, CUDA context warmed, no
cubin cache) of es_check per config, default latency policy."""
import json, os, sys, time
sys.path.insert(0, '.')
import bench
from paper_2512_06627_b200 import es, shard

shard.alu_peak(0)  # CUDA context + module load outside the timed call
name = sys.argv[1] if len(sys.argv) > 1 else "mult16"
x, _ = bench.build_workload(name)
t = time.perf_counter()
r = es.es_check(bench._Sub(x))
ms = 1e3 * (time.perf_counter() - t)
print(json.dumps({"config": name, "verdict": r.verdict, "cold_ms": round(ms, 1), **{k: r.stats.get(k) for k in ("engine", "jit_ms", "device_ms", "jit_opt", "cofactor_pis")}}))
