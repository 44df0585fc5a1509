"""Dev probe: split K1 build (es_split.cpp) -- cold JIT time, sweep time and
verdict per phase count, one fresh process per setting (ES_JIT_CACHE=0).

    python scripts/probe_split.py            # driver: runs every setting
    python scripts/probe_split.py one <miter> <k> <parts>
"""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(name, k, parts):
    from paper_2512_06627_b200 import miter as M, es
    m = M.gen_multiplier_miter(16, "array", "booth")
    if name == "fault":
        m = M.flip_gate(m, 1953)
    p = es.compile_program(m)
    t = time.perf_counter()
    r = es.run_exhaustive(p, engine="jit", cofactor=k if k else "none", jit_parts=parts)
    wall = (time.perf_counter() - t) * 1e3
    dev = [es.run_exhaustive(p, engine="jit", cofactor=k if k else "none", jit_parts=parts).stats["device_ms"]
           for _ in range(3)]
    s = r.stats
    print(json.dumps({"miter": name, "k": k, "parts": parts, "verdict": r.verdict, "witness": r.witness_index,
                      "cold_wall_ms": round(wall, 1), "jit_ms": round(s["jit_ms"], 1),
                      "compile_ms": round(s["compile_ms"], 1), "cold_device_ms": round(s["device_ms"], 2),
                      "device_ms": round(min(dev), 3), "regs": s["regs_per_thread"], "jit_parts": s["jit_parts"],
                      "jit_opt": s["jit_opt"]}), flush=True)


def auto(name):
    from paper_2512_06627_b200 import miter as M, es
    m = M.gen_multiplier_miter(16, "array", "booth")
    if name == "fault":
        m = M.flip_gate(m, 1953)
    for i in range(4):
        t = time.perf_counter()
        r = es.es_check(_Sub(m))
        wall = (time.perf_counter() - t) * 1e3
        s = r.stats
        print(json.dumps({"miter": name, "run": i, "verdict": r.verdict, "wall_ms": round(wall, 1),
                          "jit_ms": round(s["jit_ms"], 1), "device_ms": round(s["device_ms"], 2),
                          "k": s["cofactor_pis"], "jit_parts": s["jit_parts"], "jit_opt": s["jit_opt"],
                          "engine": s["engine"]}), flush=True)


class _Sub:  # es_check reads .circuit (sweep.py:44-51)
    def __init__(self, circuit):
        self.circuit = circuit


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "auto":
        auto(sys.argv[2])
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
        sys.exit(0)
    env = dict(os.environ, ES_JIT_CACHE="0")
    for name in ("eq", "fault"):
        for k in (0, 2):
            for parts in (1, 2, 4, 8, 16):
                subprocess.run([sys.executable, __file__, "one", name, str(k), str(parts)], env=env)
    # the policy's own cold choice (engine auto, cofactor auto), then warm re-runs
    for name in ("eq", "fault"):
        subprocess.run([sys.executable, __file__, "auto", name], env=env)
