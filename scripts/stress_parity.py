"""Randomised parity stress (test infrastructure; GPU box): miters of random
XAGs against single-gate faults of themselves (outputs that are 1 on few,
deep patterns) and multiplier faults, checked on every engine / policy of
the product path against the oracle's canonical minimum-index witness
(oracle/es_oracle.c, workers=1 semantics).

    python scripts/stress_parity.py [n_cases] [seed] [min_pis max_pis max_gates]
"""
import json
import random
import sys
import time

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (the checker, never the product)
from paper_2512_06627_b200 import es, miter as M  # noqa: E402
from paper_2512_06627_b200.xag import XagBuilder, random_xag  # noqa: E402

# (engine, cofactor, jit_parts): the direct-SASS builds (-1) first, so no
# ptxas kernel of the same variant is cached yet (a cached higher-level kernel
# would serve the request)
MODES = [("jit", "none", -1), ("jit", 2, -1), ("jit", 4, -1),
         ("interp", "none", 0), ("interp", "auto", 0), ("interp", "throughput", 0),
         ("jit", "none", 0), ("jit", "auto", 0), ("jit", "throughput", 0), ("jit", 2, 0), ("jit", 4, 0)]


def cases(n, seed, lo=12, hi=27, max_gates=500):
    rng = random.Random(seed)
    for k in range(n):
        if k % 5 == 4:
            w = rng.choice([6, 8, 10])
            m = M.gen_multiplier_miter(w, "array", rng.choice(["booth", "wallace", "diagonal"]))
            yield f"mult{w}-flip", M.flip_gate(m, rng.randrange(len(m.gates)))
            continue
        n_pis = rng.randint(lo, hi)
        x = random_xag(n_pis, rng.randint(40, max_gates), seed=seed * 100003 + k)
        if not x.gates:
            continue
        # fault a gate near the output (so it usually reaches it), then gate
        # the miter with a conjunction of high PIs: the witnesses go deep
        y = M.flip_gate(x, rng.randrange(max(0, len(x.gates) - 20), len(x.gates)))
        m = M.build_miter(x, y)
        b = XagBuilder(m.num_pis)
        (o,) = M.copy_into(b, m)
        for j in rng.sample(range(max(1, n_pis - 8), n_pis + 1), rng.randint(0, 5)):
            o = b.add_and(o, b.pi(j))
        yield f"rand{n_pis}", b.finish([o])


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    lo, hi, mg = (int(a) for a in sys.argv[3:6]) if len(sys.argv) > 5 else (12, 27, 500)
    t0 = time.time()
    stats = {"cases": 0, "runs": 0, "eq": 0, "neq": 0, "mismatches": []}
    for name, x in cases(n, seed, lo, hi, mg):
        if x.num_pis > 40:
            continue
        ref_v, ref_w, _ = O.min_witness(O.compile_program(x))
        p = es.compile_program(x)
        stats["cases"] += 1
        stats["eq" if ref_w is None else "neq"] += 1
        for engine, cof, parts in MODES:
            if engine == "jit" and x.num_pis < 6:
                continue
            r = es.run_exhaustive(p, engine=engine, cofactor=cof, jit_parts=parts)
            stats["runs"] += 1
            if parts == -1 and r.stats["jit_parts"] == -1:
                stats["direct_runs"] = stats.get("direct_runs", 0) + 1
            if r.witness_index != ref_w:
                stats["mismatches"].append([name, x.num_pis, len(x.gates), engine, str(cof), parts,
                                            r.verdict, r.witness_index, ref_w])
    stats["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(stats))
    sys.exit(1 if stats["mismatches"] else 0)


if __name__ == "__main__":
    main()
