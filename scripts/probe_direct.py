"""Dev probe: direct-SASS K1 (es_sass.cpp) vs ptxas builds on mult16 and the
config-5 fault miter: cold wall time (fresh process, no disk cache), JIT time
and warm device time per build.
    python scripts/probe_direct.py            # driver: one process per setting
    python scripts/probe_direct.py one <miter> <cofactor> <jit_parts>
"""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(name, cof, parts):
    from paper_2512_06627_b200 import miter as M, es
    m = M.gen_multiplier_miter(16, "array", "booth")
    if name == "fault":
        m = M.flip_gate(m, 1953)
    cof = cof if cof in ("auto", "none", "throughput") else int(cof)
    t = time.perf_counter()
    p = es.compile_program(m)
    r = es.run_exhaustive(p, engine="jit", cofactor=cof, jit_parts=parts)
    wall = (time.perf_counter() - t) * 1e3
    dev = [es.run_exhaustive(p, engine="jit", cofactor=cof, jit_parts=parts).stats["device_ms"] for _ in range(5)]
    s = r.stats
    print(json.dumps({"miter": name, "cofactor": cof, "jit_parts": parts, "verdict": r.verdict,
                      "witness": r.witness_index, "cold_wall_ms": round(wall, 2), "jit_ms": round(s["jit_ms"], 2),
                      "cold_device_ms": round(s["device_ms"], 3), "warm_device_ms": round(min(dev), 4),
                      "build": s["jit_parts"], "k": s["cofactor_pis"], "regs": s["regs_per_thread"],
                      "phases": s["phases"]}), flush=True)


def auto(name):
    from paper_2512_06627_b200 import miter as M, es
    m = M.gen_multiplier_miter(16, "array", "booth")
    if name == "fault":
        m = M.flip_gate(m, 1953)
    for i in range(4):
        t = time.perf_counter()
        r = es.run_exhaustive(es.compile_program(m))
        wall = (time.perf_counter() - t) * 1e3
        s = r.stats
        print(json.dumps({"miter": name, "mode": "auto", "run": i, "verdict": r.verdict, "witness": r.witness_index,
                          "wall_ms": round(wall, 2), "jit_ms": round(s["jit_ms"], 2), "device_ms": round(s["device_ms"], 3),
                          "build": s["jit_parts"], "k": s["cofactor_pis"], "phases": s["phases"]}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one(sys.argv[2], sys.argv[3], int(sys.argv[4]))
    elif len(sys.argv) > 1 and sys.argv[1] == "auto":
        auto(sys.argv[2])
    else:
        env = dict(os.environ, ES_JIT_CACHE="0")
        runs = [("mult16", c, p) for c in ("none", "2", "4") for p in (-1, 1)] + \
               [("fault", c, p) for c in ("none", "4") for p in (-1,)]
        for name, c, p in runs:
            subprocess.run([sys.executable, __file__, "one", name, c, str(p)], env=env, timeout=300)
        for name in ("mult16", "fault"):
            subprocess.run([sys.executable, __file__, "auto", name], env=env, timeout=300)
