"""On-disk cubin cache (es_jit.cpp; the reference's numba cache=True): a
second process loads the first process's cubins instead of running ptxas,
and gets the same verdict.  (Direct-SASS builds, es_sass.cpp, take ~6 ms and
are not cached on disk; the test forces a ptxas build.)"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = """
import sys, json; sys.path.insert(0, %r)
from paper_2512_06627_b200 import es, miter as M
m = M.flip_gate(M.gen_multiplier_miter(10, "array", "booth"), 400)
r = es.run_exhaustive(es.compile_program(m), engine="jit", cofactor=2, jit_parts=1)  # a ptxas build
print(json.dumps({"jit_ms": r.stats["jit_ms"], "verdict": r.verdict, "w": r.witness_index}))
""" % ROOT


@pytest.mark.gpu
def test_second_process_skips_ptxas(tmp_path, gpu):
    env = dict(os.environ, ES_JIT_CACHE="1", ES_JIT_CACHE_DIR=str(tmp_path))
    runs = []
    for _ in range(2):
        r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        runs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert any(p.suffix == ".esbin" for p in tmp_path.iterdir())
    assert (runs[0]["verdict"], runs[0]["w"]) == (runs[1]["verdict"], runs[1]["w"])
    assert runs[1]["jit_ms"] < 0.5 * runs[0]["jit_ms"]


@pytest.mark.gpu
def test_cache_off_and_corrupt_entries(tmp_path, gpu):
    env = dict(os.environ, ES_JIT_CACHE="0", ES_JIT_CACHE_DIR=str(tmp_path))
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and not list(tmp_path.iterdir())
    env["ES_JIT_CACHE"] = "1"
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
    ref = json.loads(r.stdout.strip().splitlines()[-1])
    for p in tmp_path.iterdir():  # truncate every entry: must recompile, not crash
        p.write_bytes(p.read_bytes()[:40])
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert (got["verdict"], got["w"]) == (ref["verdict"], ref["w"])


LEVELS = """
import sys, json; sys.path.insert(0, %r)
from paper_2512_06627_b200 import es, miter as M
m = M.flip_gate(M.gen_multiplier_miter(10, "array", "booth"), 400)
p = es.compile_program(m)
out = []
for cof in ("auto", "throughput", "none"):
    r = es.run_exhaustive(p, engine="jit", cofactor=cof)
    out.append([cof, r.stats["jit_opt"], r.verdict, r.witness_index])
print(json.dumps(out))
""" % ROOT


@pytest.mark.gpu
def test_cold_runs_build_direct_throughput_at_o3(gpu):
    """A cold latency-mode run is JIT-bound: the policy writes the kernel's
    SASS directly (es_sass.cpp, build level 0, no ptxas); throughput mode
    compiles at ptxas -O3.  Same verdict and minimum-index witness either way."""
    env = dict(os.environ, ES_JIT_CACHE="0")
    env.pop("ES_PTXAS_O", None)
    r = subprocess.run([sys.executable, "-c", LEVELS], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    runs = json.loads(r.stdout.strip().splitlines()[-1])
    levels = {cof: opt for cof, opt, _, _ in runs}
    assert levels["auto"] == 0 and levels["throughput"] == 3
    assert len({(v, w) for _, _, v, w in runs}) == 1 and runs[0][2] == "COUNTEREXAMPLE"
