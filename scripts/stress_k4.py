"""Stress parity for K4: batches of 18-24-PI cones cut from clean and faulty
multiplier / adder miters (the sweep's own candidate pairs), each run with
K4 (engine auto) and with the K2 interpreter alone (pinned to the oracle by
tests/test_config4_gpu.py and scripts/stress_parity.py); verdict, witness
and patterns_evaluated must be equal job for job (the library also
re-checks every witness on its sub-miter)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2512_06627_b200 import cones, miter as M

t0 = time.time()
cases = []
for w, a, b in [(10, "array", "booth"), (10, "array", "wallace"), (12, "array", "booth"), (12, "array", "wallace")]:
    base = M.gen_multiplier_miter(w, a, b)
    cases.append((f"mult{w}-{b}", base))
    for f in (97, 211, 333, 517, 801):
        if f < len(base.gates):
            cases.append((f"mult{w}-{b}-f{f}", M.flip_gate(base, f)))
jobs = mism = k4jobs = cex = 0
for name, m in cases:
    bt = cones.sweep_round_batch(m, lo=18, hi=24)
    if len(bt) == 0:
        continue
    bt.select(list(range(min(len(bt), 300))))
    r4 = bt.run_arrays()
    r2 = bt.run_arrays(engine="interp")
    r4b = bt.run_arrays()
    bad = [i for i in range(len(bt)) if any(r4[k][i] != r2[k][i] or r4b[k][i] != r2[k][i]
                                            for k in ("verdict", "witness_index", "patterns_evaluated"))]
    jobs += len(bt); mism += len(bad); k4jobs += int((r4["engine"] == 1).sum()); cex += int((r2["verdict"] == 1).sum())
    print(f"{name}: jobs={len(bt)} k4={int((r4['engine'] == 1).sum())} cex={int((r2['verdict'] == 1).sum())} mismatches={len(bad)}", flush=True)
print(f"TOTAL jobs={jobs} k4_jobs={k4jobs} cex={cex} mismatches={mism} in {time.time() - t0:.0f} s", flush=True)
assert mism == 0
