"""Dev probe: where the COLD GPU sweep of the 16x16 array-vs-Booth miter
spends its wall time (first sweep in the process, cProfile)."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.sweep import SweepConfig, sweep
from paper_2512_06627_b200 import es
x = M.gen_multiplier_miter(16, "array", "booth")
es.compile_program(M.gen_multiplier_miter(4, "array", "booth"))  # library + context warm
es.run_exhaustive(es.compile_program(M.gen_multiplier_miter(4, "array", "booth")))
t = time.perf_counter()
cProfile.run("r = sweep(x, SweepConfig())", "/tmp/sw.prof")
print("cold sweep", round((time.perf_counter() - t) * 1e3, 1), "ms", r.verdict,
      {k: r.stats.get(k) for k in ("rounds", "engine_calls", "merges")})
pstats.Stats("/tmp/sw.prof").sort_stats("cumulative").print_stats(14)
