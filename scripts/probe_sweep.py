"""Dev probe: the GPU sweep (engine es) on the config multiplier miters."""
import sys, time
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200.sweep import SweepConfig, sweep
for w, a, b in [(12, "array", "wallace"), (16, "array", "booth"), (12, "array", "wallace"), (16, "array", "booth")]:
    x = M.gen_multiplier_miter(w, a, b)
    t = time.time(); r = sweep(x, SweepConfig()); dt = time.time() - t
    print(w, a, b, r.verdict, round(dt, 3), r.engine, {k: r.stats.get(k) for k in ("engine_calls", "merges", "structural_merges", "refinements", "rounds", "unknown_pairs", "device_ms", "jit_ms")}, flush=True)
