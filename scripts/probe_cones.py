"""Dev probe: config-4 batch (10k cones) device / wall time under the K2
knobs in the environment (ES_K2_CTAS, ES_K2_MAXSLOTS)."""
import os, sys, time
sys.path.insert(0, '.')
from paper_2512_06627_b200 import cones
t = time.time(); b = cones.config4_batch(10000); tb = time.time() - t
best = 1e9
for i in range(4):
    t = time.time(); r = b.run_arrays(); w = time.time() - t
    best = min(best, float(r["device_ms"].max()))
print(f"CTAS={os.environ.get('ES_K2_CTAS', '-')} MAXSLOTS={os.environ.get('ES_K2_MAXSLOTS', '-')} "
      f"build={tb:.1f}s device={best:.2f}ms wall={w * 1e3:.1f}ms", flush=True)
