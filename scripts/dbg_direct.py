import sys; sys.path.insert(0,'.')
from paper_2512_06627_b200 import es, miter as M
p = es.compile_program(M.gen_multiplier_miter(8,'array','booth'))
k = sys.argv[1]
r = es.run_exhaustive(p, engine="jit", cofactor=("none" if k=='0' else int(k)), jit_parts=-1)
print('k', k, r.verdict, r.stats['jit_parts'], r.stats['device_ms'])
