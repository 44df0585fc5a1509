import sys; sys.path.insert(0,'.')
from paper_2512_06627_b200 import miter as M, es
m = M.gen_multiplier_miter(16, "array", "booth")
p = es.compile_program(m)
for k in (3, 4):
    for bt in (128, 256):
        ts = [es.run_exhaustive(p, engine="jit", cofactor=k, block_threads=bt).stats for _ in range(6)]
        print(k, bt, min(t["device_ms"] for t in ts[2:]), ts[-1]["regs_per_thread"], flush=True)
