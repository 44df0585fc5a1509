"""Dev probe: K4 on the sweep's own batches -- the 192-cone EQ-heavy round
(cones.sweep_round_batch, cold first run and warm) and whole sweeps of the
config multiplier miters (cold = first in the process, then warm)."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2512_06627_b200 import cones, miter as M
from paper_2512_06627_b200.sweep import SweepConfig, sweep

tag = f"K4={os.environ.get('ES_K4', '1')}"
b = cones.sweep_round_batch()
ts, dv = [], []
for rep in range(5):
    t = time.perf_counter()
    rec = b.run_arrays()
    ts.append((time.perf_counter() - t) * 1e3)
    dv.append(float(rec["device_ms"].max()))
print(f"{tag} eq-round jobs={len(b)} eq={int((rec['verdict'] == 0).sum())} engines={np.bincount(rec['engine'], minlength=3).tolist()} "
      f"API first {ts[0]:.1f} best {min(ts[1:]):.2f} ms, device first {dv[0]:.2f} best {min(dv[1:]):.2f} ms", flush=True)
for w, a, bb in [(12, "array", "wallace"), (16, "array", "booth")]:
    x = M.gen_multiplier_miter(w, a, bb)
    t = time.perf_counter(); r = sweep(x, SweepConfig()); cold = time.perf_counter() - t
    reps = []
    for _ in range(3):
        t = time.perf_counter(); sweep(x, SweepConfig()); reps.append(time.perf_counter() - t)
    print(f"{tag} sweep mult{w}: {r.verdict} cold {cold * 1e3:.0f} ms warm {min(reps) * 1e3:.0f} ms", flush=True)
