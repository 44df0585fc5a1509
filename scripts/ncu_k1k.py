"""ncu target: mult16 K1 at a forced cofactor depth (argv[1]), three verdicts."""
import sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import es, miter as M
p = es.compile_program(M.gen_multiplier_miter(16, "array", "booth"))
k = int(sys.argv[1])
for v in range(3):
    es.run_exhaustive(p, engine="jit", cofactor=k, jit_parts=int(sys.argv[2]) if len(sys.argv) > 2 else 1)
