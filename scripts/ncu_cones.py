"""ncu target: the config-4 batch (10k cones), one batched K2 verdict."""
import sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import cones
b = cones.config4_batch(10000)
b.run_arrays()
