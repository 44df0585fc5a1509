"""Dev probe: K1 variants on mult16 (EQ) and the config-5 fault miter, one
process per setting, knobs from the environment (ES_K1_SPILL_R, ES_MAXNREG,
ES_IMAD_COST, ...).  Prints device time and verdict parity.
    ES_K1_SPILL_R=140 ES_MAXNREG=168 python scripts/probe_k1var.py 4 128
"""
import os, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import miter as M, es

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
bt = int(sys.argv[2]) if len(sys.argv) > 2 else 256
tag = " ".join(f"{v}={os.environ[v]}" for v in ("ES_K1_SPILL_R", "ES_MAXNREG", "ES_IMAD_COST") if v in os.environ)
circ = sys.argv[3] if len(sys.argv) > 3 else "mult16"
if circ == "mult16":
    m = M.gen_multiplier_miter(16, "array", "booth")
    cases = (("mult16", m, None), ("fault1953", M.flip_gate(m, 1953), 1610645504))
else:  # a butterfly network with a ~512-value live set (tests/wide_circuits.py), EQ
    sys.path.insert(0, "tests")
    import wide_circuits as W
    cases = (("bfly32", W.butterfly(32, 256, 8, eq=True), None),)
for name, x, want in cases:
    p = es.compile_program(x)
    ts = []
    for rep in range(6 if want is None else 3):
        r = es.run_exhaustive(p, engine="jit", cofactor=k, jit_parts=1, block_threads=bt)
        ts.append(r.stats['device_ms'])
    ok = (r.verdict == es.EXHAUSTED_ZERO) if want is None else (r.witness_index == want)
    t = min(ts[1:])
    print(f"{tag} k={k} T={bt} {name}: dev={t:.4f}ms med={sorted(ts[1:])[len(ts[1:]) // 2]:.4f} "
          f"rate={p.num_gates * 2**32 / (t * 1e-3):.3e} ok={ok} regs={r.stats.get('regs_per_thread')} "
          f"jit={r.stats.get('jit_ms'):.0f}", flush=True)
