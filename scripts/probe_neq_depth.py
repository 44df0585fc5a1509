"""Time-to-verdict of a non-equivalent 32-PI miter against witness depth
(VERDICT r01 next #4): the mult16 array-vs-Booth miter with ONE failing
pattern ORed in at a chosen index, for every K1 cofactor depth and the
throughput policy (two-phase search).  Warm: the kernels are compiled by an
untimed run first.  Writes the table as JSON (profiles/r02_neq_depth.json).

    python scripts/probe_neq_depth.py [out.json]
"""
import json
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2512_06627_b200 import es  # noqa: E402
from tests.golden import recipes  # noqa: E402

DEPTHS = [1 << 20, 1 << 24, (1 << 28) + 1, 1610645504, 3 << 29, 1 << 31, (1 << 32) - 1]
MODES = ["none", 1, 2, 3, 4, "throughput"]


def main(out_path):
    eq = es.compile_program(recipes.build_sweep_circuit({"kind": "mult", "width": 16, "a": "array",
                                                         "b": "booth"}))
    rows = []
    ref = {}
    for mode in MODES:
        es.run_exhaustive(eq, engine="jit", cofactor=mode)
        d = [es.run_exhaustive(eq, engine="jit", cofactor=mode).stats["device_ms"] for _ in range(5)]
        ref[str(mode)] = statistics.median(d)
    for needle in DEPTHS:
        x = recipes.build_sweep_circuit({"kind": "mult", "width": 16, "a": "array", "b": "booth",
                                         "needle": needle})
        p = es.compile_program(x)
        for mode in MODES:
            r = es.run_exhaustive(p, engine="jit", cofactor=mode)  # JIT (both phases)
            assert r.witness_index == needle, (needle, mode, r.witness_index)
            devs, walls = [], []
            for _ in range(5):
                t = time.perf_counter()
                r = es.run_exhaustive(p, engine="jit", cofactor=mode)
                walls.append(1e3 * (time.perf_counter() - t))
                devs.append(r.stats["device_ms"])
            row = {"witness": needle, "depth_frac": needle / 2 ** 32, "mode": str(mode),
                   "device_ms": statistics.median(devs), "wall_ms": statistics.median(walls),
                   "eq_sweep_ms": ref[str(mode)], "vs_eq_same_mode": statistics.median(devs) / ref[str(mode)],
                   "vs_eq_throughput": statistics.median(devs) / ref["throughput"],
                   "cofactor_pis": r.stats["cofactor_pis"], "phases": r.stats["phases"],
                   "phase2_cofactor_pis": r.stats["phase2_cofactor_pis"],
                   "patterns_swept_frac": r.stats["patterns_swept"] / 2 ** 32}
            rows.append(row)
            print(json.dumps(row), flush=True)
    json.dump({"workload": "mult16 array-vs-Booth + one failing minterm at `witness` (32 PIs)",
               "eq_sweep_ms": ref, "rows": rows}, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/neq_depth.json")
