"""ncu target: K2 interpreter on mult12 (single job) then the config-4 batch."""
import sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import es, miter as M, cones
p = es.compile_program(M.gen_multiplier_miter(12, "array", "wallace"))
for _ in range(3):
    es.run_exhaustive(p, engine="interp")
b = cones.config4_batch(10000)
b.run()
