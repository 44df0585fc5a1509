"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every fixture row is produced by the reference package (cecprove): its
``compile_program`` (es.py:87) and ``run_exhaustive(workers=1)`` (es.py:252),
plus ``truth_table``/``first_one_row`` (eval.py:69-92) where <= 22 PIs.  The
circuits are rebuilt from seeds/recipes by this repo's generators; the fixture
stores a hash of each circuit, and the make step asserts that the reference's
own generators (random_xag, gen_multiplier_miter, mutate, build_miter) give
the identical circuit wherever the reference has one.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from cecprove import es as ref_es  # noqa: E402  (reference, read-only)
from cecprove import eval as ref_eval  # noqa: E402
from cecprove import miter as ref_miter  # noqa: E402
from cecprove import xag as ref_xag  # noqa: E402

from tests.golden import recipes  # noqa: E402


def to_ref(x):
    return ref_xag.Xag(x.num_pis,
                       tuple(ref_xag.Gate(ref_xag.GateKind(int(g.kind)),
                                          ref_xag.Lit(g.in0.node, bool(g.in0.neg)),
                                          ref_xag.Lit(g.in1.node, bool(g.in1.neg)))
                             for g in x.gates),
                       tuple(ref_xag.Lit(o.node, bool(o.neg)) for o in x.outputs))


def ref_prog_rows(p):
    return [[i.op, i.dst, i.src0, int(i.neg0), i.src1, int(i.neg1), i.pi] for i in p.instrs]


def row(x, ref_x=None, full_program=False, workers=1):
    if ref_x is not None:
        assert recipes.xag_sha(ref_x) == recipes.xag_sha(x), "generator drift vs reference"
    rx = to_ref(x)
    t0 = time.monotonic()
    try:
        p = ref_es.compile_program(rx)
    except ref_es.TooManyInputs:
        return {"xag_sha": recipes.xag_sha(x), "too_many_inputs": True}
    rows = ref_prog_rows(p)
    r = ref_es.run_exhaustive(p, workers=workers)
    dt = time.monotonic() - t0
    widx = None
    if r.witness is not None:
        widx = sum(b << i for i, b in enumerate(r.witness))
    out = {
        "xag_sha": recipes.xag_sha(x),
        "num_pis": x.num_pis,
        "num_gates": len(x.gates),
        "prog_sha": recipes.prog_sha(rows, p.num_registers),
        "num_instrs": len(rows),
        "num_registers": p.num_registers,
        "G": sum(1 for q in rows if q[0] in (1, 2)),
        "verdict": r.verdict,
        "witness_index": widx,
        "patterns_evaluated": r.patterns_evaluated,
        "ref_workers": workers,
        "ref_seconds": round(dt, 4),
    }
    if x.num_pis <= 22 and workers == 1:
        tt = ref_eval.truth_table(rx)
        first = ref_eval.first_one_row(tt, x.num_pis)
        tt_idx = None if first is None else sum(b << i for i, b in enumerate(first))
        # the survey's claim: workers=1 witness == truth-table lowest row
        assert tt_idx == widx, (tt_idx, widx)
    if full_program:
        out["program"] = rows
    return out


def cone_rows(limit: int = 240):
    """Config-4 fixtures: sub-miters cut by the REFERENCE's extract_submiter
    (sweep.py:92-158) for candidate pairs of the array-vs-Booth 16x16 miter."""
    from cecprove import sweep as ref_sweep
    from paper_2512_06627_b200 import cones

    m, pairs = next(cones.config4_pairs())
    rm = to_ref(m)
    rows = []
    for k, (a, b, pol) in enumerate(pairs[:limit]):
        sm = ref_sweep.extract_submiter(rm, a, b, {}, polarity=pol, sm_id=k)
        r = row(sm.circuit)
        r.update({"pair": [a, b, int(pol)], "pi_map": list(sm.pi_map)})
        rows.append(r)
    return rows


def main() -> None:
    t_start = time.monotonic()
    fixtures: dict[str, list] = {}
    path = os.path.join(HERE, "golden.json")
    if "--only-cones" in sys.argv:
        doc = json.load(open(path))
        doc["fixtures"]["cones"] = cone_rows()
        with open(path, "w") as fh:
            json.dump(doc, fh, separators=(",", ":"))
        print(f"cones: {len(doc['fixtures']['cones'])} rows, {time.monotonic() - t_start:.1f}s")
        return

    # 1. random XAG populations of the reference's own tests
    rand_rows = []
    for spec in recipes.random_population():
        x = recipes.build_random(spec)
        ref_x = ref_xag.random_xag(spec["n_pis"], spec["n_gates"], spec["seed"])
        r = row(x, ref_x)
        r.update(spec)
        rand_rows.append(r)
    fixtures["random"] = rand_rows
    print(f"random: {len(rand_rows)} rows, {time.monotonic() - t_start:.1f}s", flush=True)

    # 2. named miters and mutants
    miter_rows = []
    for spec in recipes.miter_population():
        x = recipes.build_miter_recipe(spec)
        ref_x = recipes.build_with_reference(spec, ref_miter, ref_xag)
        r = row(x, ref_x, full_program=spec.get("full_program", False),
                workers=spec.get("ref_workers", 1))
        r.update(spec)
        miter_rows.append(r)
        print(f"  {spec['name']}: {r['verdict']} idx={r.get('witness_index')} "
              f"G={r.get('G')} {r.get('ref_seconds')}s", flush=True)
    fixtures["miters"] = miter_rows
    fixtures["cones"] = cone_rows()

    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "cecprove (arxiv 2512.06627 package) es.py/eval.py",
                   "fixtures": fixtures}, fh, separators=(",", ":"))
    print(f"done in {time.monotonic() - t_start:.1f}s")


if __name__ == "__main__":
    main()
