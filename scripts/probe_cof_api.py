"""Dev probe: K1 cofactor depths on the config miters through the engine API."""
import json, sys
sys.path.insert(0, '.')
from paper_2512_06627_b200 import es
from tests.golden import recipes
gold = {r["name"]: r for r in json.load(open("tests/golden/golden.json"))["fixtures"]["miters"]}
specs = {s["name"]: s for s in recipes.miter_population()}
names = sys.argv[1:] or ["mult16_array_booth", "mult16_array_booth_flip1953", "mult14_array_booth"]
for name in names:
    x = recipes.build_miter_recipe(specs[name]); g = gold[name]
    p = es.compile_program(x)
    for bt in (128, 256):
        for cof in (0, 1, 2, 3, 4, "throughput", "auto"):
            ts, jit = [], 0
            for rep in range(6):
                r = es.run_exhaustive(p, engine="jit", cofactor=cof, block_threads=bt)
                ts.append(r.stats["device_ms"]); jit = max(jit, r.stats["jit_ms"])
            ok = r.verdict == g["verdict"] and r.witness_index == g["witness_index"]
            t = min(ts[1:])
            W = p.num_gates * 2 ** x.num_pis
            print(f"{name:30s} bt={bt} cof={str(cof):10s} k={r.stats['cofactor_pis']} ok={ok} dev={t:7.3f}ms "
                  f"EQ-rate={W / (t * 1e-3):.3e} luts={r.stats['luts']} regs={r.stats['regs_per_thread']} "
                  f"jit={jit:.0f}ms compile={r.stats['compile_ms']:.1f}ms", flush=True)
