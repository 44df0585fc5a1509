"""ncu target: the bench's K1 kernel (mult16 array-vs-Booth, throughput mode:
4 cofactor PIs), three verdicts."""
import sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import es, miter as M
p = es.compile_program(M.gen_multiplier_miter(16, "array", "booth"))
for v in range(3):
    es.run_exhaustive(p, engine="jit", cofactor="throughput")
