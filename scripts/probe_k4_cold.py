"""Dev probe: where a cold K4 run's time goes (ES_VERBOSE=1 prints the
library's breakdown): CUDA init, batch build, prepare, first and second run."""
import os, sys, time
sys.path.insert(0, '.')
t0 = time.perf_counter()
from paper_2512_06627_b200 import cones, es, miter as M
import torch
x = M.gen_multiplier_miter(8, "array", "booth")
es.run_exhaustive(es.compile_program(x))  # CUDA context + library init
t1 = time.perf_counter()
b = cones.sweep_round_batch()
t2 = time.perf_counter()
b.prepare()
t3 = time.perf_counter()
for i in range(3):
    t = time.perf_counter()
    rec = b.run_arrays()
    print(f"run {i}: {(time.perf_counter() - t) * 1e3:.1f} ms device {float(rec['device_ms'].max()):.2f}", flush=True)
print(f"init {(t1 - t0) * 1e3:.0f} ms, batch {(t2 - t1) * 1e3:.0f} ms, prepare {(t3 - t2) * 1e3:.0f} ms", flush=True)
