"""Dev probe: config 4 (10,000 cones) with K4 (straight-line bodies in
multi-body modules) against the K2-only run of the same batch: verdicts,
witnesses and patterns_evaluated equal, device and API times.  One process
per setting (ES_K4, ES_K4_MIN_PIS are read once):
    ES_K4_MIN_PIS=20 python scripts/probe_k4.py
"""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2512_06627_b200 import cones

b = cones.config4_batch(10_000)
t = time.perf_counter()
b.prepare()
prep_ms = (time.perf_counter() - t) * 1e3
ref = b.run_arrays(engine="interp")
keys = ("verdict", "witness_index", "patterns_evaluated")
dev, api = [], []
for rep in range(5):
    t = time.perf_counter()
    rec = b.run_arrays()
    api.append((time.perf_counter() - t) * 1e3)
    dev.append(float(rec["device_ms"].max()))
    bad = [i for i in range(len(rec)) if any(rec[k][i] != ref[k][i] for k in keys)]
    assert not bad, (len(bad), bad[:5], [(rec[i], ref[i]) for i in bad[:2]])
eng = np.bincount(rec["engine"], minlength=3)
print(f"K4={os.environ.get('ES_K4', '1')} min_pis={os.environ.get('ES_K4_MIN_PIS', '20')} "
      f"device first {dev[0]:.2f} best {min(dev[1:]):.2f} ms | API first {api[0]:.1f} best {min(api[1:]):.1f} ms "
      f"| prepare {prep_ms:.0f} ms | engines {eng.tolist()} | interp-only device {float(ref['device_ms'].max()):.2f} ms", flush=True)
