"""Dev probe: where the GPU sweep's wall time goes (cProfile); argv[1] =
multiplier width (array vs Wallace), ES_VERBOSE=1 for per-batch timing."""
import cProfile, pstats, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.sweep import SweepConfig, sweep
w = int(sys.argv[1]) if len(sys.argv) > 1 else 12
x = M.gen_multiplier_miter(w, "array", "wallace")
sweep(x, SweepConfig())
cProfile.run("r = sweep(x, SweepConfig())", "/tmp/sw.prof")
print(r.verdict, {k: r.stats.get(k) for k in ("rounds", "engine_calls", "merges", "wall_time")})
pstats.Stats("/tmp/sw.prof").sort_stats("cumulative").print_stats(8)
