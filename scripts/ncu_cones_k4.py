"""ncu target: config 4 (10,000 cones) batched verdict, twice (the second
run is warm: K4 modules loaded, images resident)."""
import sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import cones
b = cones.config4_batch(10_000)
for _ in range(2):
    b.run_arrays()
