"""Dev probe: where the GPU sweep's wall time goes (cProfile)."""
import cProfile, pstats, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.sweep import SweepConfig, sweep
x = M.gen_multiplier_miter(12, "array", "wallace")
sweep(x, SweepConfig())
cProfile.run("sweep(x, SweepConfig())", "/tmp/sw.prof")
pstats.Stats("/tmp/sw.prof").sort_stats("cumulative").print_stats(18)
