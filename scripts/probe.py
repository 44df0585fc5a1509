"""Quick GPU probe: parity on the config miters + timings (dev tool)."""
import sys, time, json
sys.path.insert(0, '.')
import __graft_entry__ as ge
ge.build(); ge.smoke()
from paper_2512_06627_b200 import es, miter as M
from tests.golden import recipes
from oracle import oracle as O
gold = {r["name"]: r for r in json.load(open("tests/golden/golden.json"))["fixtures"]["miters"]}
specs = {s["name"]: s for s in recipes.miter_population()}
for name in ["adder8_ripple_lookahead", "mult12_array_wallace", "mult12_array_wallace_flip1108",
             "mult14_array_booth", "mult16_array_booth", "mult16_array_booth_flip1953",
             "mult16_array_booth_flip2204", "mult16_array_booth_flip1220"]:
    x = recipes.build_miter_recipe(specs[name]); g = gold[name]
    p = es.compile_program(x)
    for eng in ("jit", "interp") if x.num_pis <= 24 else ("jit",):
        for rep in range(3):
            t = time.perf_counter(); r = es.run_exhaustive(p, engine=eng); dt = time.perf_counter() - t
        ok = r.verdict == g["verdict"] and r.witness_index == g["witness_index"] and r.patterns_evaluated == g["patterns_evaluated"]
        W = p.num_gates * (2 ** x.num_pis if r.witness_index is None else r.stats["patterns_swept"])
        print(f"{name:34s} {eng:6s} ok={ok} {r.verdict:15s} idx={r.witness_index} wall={dt*1e3:8.2f}ms dev={r.stats['device_ms']:8.2f}ms "
              f"jit={r.stats['jit_ms']:.1f}ms luts={r.stats['luts']} regs={r.stats['regs_per_thread']} "
              f"rate={W/(r.stats['device_ms']*1e-3+1e-12):.3e} gate-pat/s", flush=True)
