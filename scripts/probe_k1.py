"""Compare K1 skeleton variants on the config miters (dev tool)."""
import sys, time, json
sys.path.insert(0, '.')
from paper_2512_06627_b200 import es
from tests.golden import recipes
gold = {r["name"]: r for r in json.load(open("tests/golden/golden.json"))["fixtures"]["miters"]}
specs = {s["name"]: s for s in recipes.miter_population()}
for name in ["mult12_array_wallace", "mult12_array_wallace_flip1108", "mult14_array_booth", "mult16_array_booth",
             "mult16_array_booth_flip1953", "mult16_array_booth_flip2204", "mult14_array_diagonal"]:
    x = recipes.build_miter_recipe(specs[name]); g = gold[name]
    p = es.compile_program(x)
    for var in sys.argv[1:] or ["k1", "k1t"]:
        ts = []
        for rep in range(5):
            r = es.run_exhaustive(p, engine="jit", variant=var)
            ts.append(r.stats['device_ms'])
        ok = r.verdict == g["verdict"] and r.witness_index == g["witness_index"] and r.patterns_evaluated == g["patterns_evaluated"]
        W = p.num_gates * (2 ** x.num_pis if r.witness_index is None else r.patterns_evaluated)
        print(f"{name:32s} {var:4s} ok={ok} dev={min(ts):8.3f}ms rate={W/(min(ts)*1e-3):.3e} regs={r.stats['regs_per_thread']} jit={r.stats['jit_ms']:.0f}ms", flush=True)
