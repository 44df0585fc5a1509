#!/usr/bin/env python
"""Benchmark of the B200 exact-simulation (ES) engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config mult16|mult12|adder8|mult16_neq|cones]

One step = one exact-simulation verdict of the configured miter: all 2^n
primary-input patterns swept (or, for a non-equivalent miter, every pattern
up to the minimum-index counterexample).  Default workload: BASELINE.json
configs[2], the 16x16 array vs radix-4 Booth multiplier miter (32 PIs, 2^32
patterns) -- the configuration BASELINE.json's metric is quoted on at
1/2/4/8 B200.

N GPUs, two launch modes (the pattern space is sharded either way):
  * ``python bench.py --gpus N`` (no torchrun): ONE es_run call drives N GPUs
    (es_run_opts.devices: one host thread per GPU, one minimum word in GPU 0's
    HBM shared as NVLink peer memory).  Fails if fewer than N GPUs are visible.
  * torchrun, one process per GPU (WORLD_SIZE must equal --gpus): each rank
    sweeps its residue class of chunks; the ranks share one minimum word over
    CUDA IPC and close every verdict with a device-side barrier
    (es_peer_arrive_wait) -- no collective and no host round trip per verdict.

Metric: simulated gate-patterns/s, gate = AND/XOR instruction of the
reference compile_program (G), so one step is G * 2^n gate-patterns of
algorithmic work.  Rank 0 prints ONE JSON line.

--impl reference runs the UNMODIFIED reference package (cecprove, installed
into baseline/_ref from /root/reference; Python + numba) through its own
public API -- run_exhaustive(compile_program(x), workers=<all host threads>,
budget=<bounded sample>) -- on the box's host cores, on the same miter.  If
baseline/_ref is missing it times the oracle's C restatement instead
(kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated gate·patterns/s and ES time-to-verdict per miter at 1/2/4/8 B200"
UNIT = "gate·patterns/s"
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


# --- workloads -------------------------------------------------------------

def build_workload(name: str):
    from paper_2512_06627_b200 import miter as M

    if name == "mult16":
        return (M.gen_multiplier_miter(16, "array", "booth"),
                "16x16 array vs radix-4 Booth multiplier miter (32 PIs, 2^32 patterns), "
                "BASELINE.json configs[2]")
    if name == "mult12":
        return (M.gen_multiplier_miter(12, "array", "wallace"),
                "12x12 array vs Wallace-tree multiplier miter (24 PIs), BASELINE.json configs[1]")
    if name == "adder8":
        return (M.gen_adder_miter(8, "ripple", "lookahead"),
                "8-bit ripple-carry vs carry-lookahead adder miter (16 PIs), BASELINE.json configs[0]")
    if name == "mult16_neq":
        m = M.gen_multiplier_miter(16, "array", "booth")
        return (M.flip_gate(m, 1953),
                "16x16 array vs Booth miter with single-gate fault (gate 1953 AND<->XOR; "
                "min-index cex 1610645504), BASELINE.json configs[4]")
    raise SystemExit(f"unknown config {name!r}")


class _Sub:
    """Minimal SubMiter stand-in (sweep.py:44-51): es_check reads .circuit."""

    def __init__(self, circuit):
        self.circuit = circuit
        self.origin = (0, 0)
        self.merged_history = {}
        self.pi_map = tuple(range(1, circuit.num_pis + 1))
        self.id = 0


# --- the reference package (baseline/_ref) ---------------------------------

_REF = None


def reference_pkg():
    """The unmodified reference (cecprove) installed in baseline/_ref, or None.
    Its numba JIT cache goes to a private temp directory."""
    global _REF
    if _REF is not None:
        return _REF or None
    _REF = False
    if not os.path.isdir(os.path.join(REF_DIR, "cecprove")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_ref_"))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import cecprove.es  # noqa: F401
        import cecprove.xag  # noqa: F401
        import cecprove

        _REF = cecprove
    except Exception as exc:  # numba missing, ...
        print(f"[bench] reference package unusable: {exc}", file=sys.stderr)
        return None
    return _REF


def to_ref(x, ref):
    """This repo's Xag as a reference Xag (field for field, xag.py:71-125)."""
    X = ref.xag
    return X.Xag(x.num_pis,
                 tuple(X.Gate(X.GateKind(int(g.kind)), X.Lit(g.in0.node, bool(g.in0.neg)),
                              X.Lit(g.in1.node, bool(g.in1.neg))) for g in x.gates),
                 tuple(X.Lit(o.node, bool(o.neg)) for o in x.outputs))


def _ref_G(p) -> int:
    return sum(1 for i in p.instrs if i.op in (1, 2))


def ref_sample(x, workers: int, seconds: float, ref=None) -> dict:
    """The reference's own run_exhaustive (es.py:252) on `workers` threads for
    at most `seconds` (its budget argument): gate-patterns/s over the patterns
    it evaluated.  A run that finishes first is a full verdict."""
    ref = ref or reference_pkg()
    p = ref.es.compile_program(to_ref(x, ref))
    G = _ref_G(p)
    ref.es.run_exhaustive(p, workers=workers, budget=0.05)  # numba JIT (cache=True) outside the timing
    t = time.perf_counter()
    r = ref.es.run_exhaustive(p, workers=workers, budget=seconds)
    dt = time.perf_counter() - t
    return {"value": G * r.patterns_evaluated / dt, "verdict": r.verdict,
            "patterns": r.patterns_evaluated, "seconds": dt, "G": G, "workers": workers,
            "witness_index": None if r.witness is None else sum(b << i for i, b in enumerate(r.witness))}


def port_sample(x, target_s: float, threads: int | None = None) -> dict:
    """The oracle's C restatement of the reference algorithm (es.py:175-339) on
    a bounded prefix of the sweep (whole 2^14-pattern batches, all threads)."""
    from oracle import oracle as O

    p = O.compile_program(x)
    G = p.num_gate_instrs
    threads = threads or os.cpu_count() or 1
    total_batches = 1 << max(x.num_pis - 14, 0)
    per_batch = 1 << min(x.num_pis, 14)
    O.min_witness(p, threads=threads, max_batches=min(total_batches, 4 * threads))  # warm-up
    probe = min(total_batches, 64 * threads)
    t = time.perf_counter()
    O.min_witness(p, threads=threads, max_batches=probe)
    dt = max(time.perf_counter() - t, 1e-6)
    nb = int(min(total_batches, max(probe, probe * target_s / dt)))
    t = time.perf_counter()
    verdict, idx, done = O.min_witness(p, threads=threads, max_batches=nb)
    dt = time.perf_counter() - t
    return {"value": G * done * per_batch / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {nb} of {total_batches} reference batches (2^{min(x.num_pis, 14)} "
                      f"patterns each) of the same sweep, G={G}, {dt:.2f}s, oracle/es_oracle.c "
                      f"(es.py:175-339 restated), {threads} threads",
            "seconds": dt}


def cpu_baseline(x, seconds: float, desc: str = "") -> dict:
    """The reference ES on the host: the better of workers=1 and workers=all
    (BASELINE.md section 4, step 3), each a bounded run; the oracle port when
    the reference package is unavailable."""
    ref = reference_pkg()
    cores = os.cpu_count() or 1
    if ref is None:
        return port_sample(x, seconds)
    one = ref_sample(x, 1, seconds / 2, ref)
    allc = ref_sample(x, cores, seconds / 2, ref)
    best = allc if allc["value"] >= one["value"] else one
    out = {"value": best["value"], "unit": UNIT, "cores": best["workers"], "kind": "reference",
           "sample": (f"cecprove.es.run_exhaustive(compile_program(x), workers={best['workers']}, "
                      f"budget={seconds / 2:.1f}s) from baseline/_ref (numba): "
                      f"{best['patterns']} patterns in {best['seconds']:.2f}s, verdict "
                      f"{best['verdict']}{desc}"),
           "workers_1": {k: one[k] for k in ("value", "patterns", "seconds", "verdict")},
           f"workers_{cores}": {k: allc[k] for k in ("value", "patterns", "seconds", "verdict")}}
    if best["verdict"] != "BUDGET_EXCEEDED":
        out["time_to_verdict_s"] = best["seconds"]
        out["witness_index"] = best["witness_index"]
    return out


# --- clocks ----------------------------------------------------------------

class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML in
    process every 2 ms, on every GPU of the run."""

    # NVML clocks-event-reason bits (nvml.h)
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40}

    def __init__(self, devices, period_s: float = 0.002):
        self.devices = list(devices) if isinstance(devices, (list, tuple)) else [devices]
        self.period = period_s
        self.samples: list[tuple[float, float, int]] = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = [pynvml.nvmlDeviceGetHandleByIndex(d) for d in sorted(set(self.devices))]
            self._max = [float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)) for h in self._h]
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nvml = None
        return self

    def _sample(self):
        nv = self._nvml
        for h, mx in zip(self._h, self._max):
            sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            try:
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
            except AttributeError:
                rs = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(h))
            self.samples.append((sm, mx, rs))

    def _run(self):
        while not self._stop.wait(self.period):
            try:
                self._sample()
            except Exception:
                return

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)
        if self._nvml is not None:
            try:
                self._sample()
            except Exception:
                pass

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": "unavailable"}
        reasons = sorted({nm for _, _, rs in self.samples for nm, bit in self.REASONS.items()
                          if rs & bit})
        return {"sm_mhz": statistics.median(sm for sm, _, _ in self.samples),
                "sm_max_mhz": max(mx for _, mx, _ in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "NVML, 2 ms period",
                "gpus": len(set(self.devices))}


# --- roofline helpers ------------------------------------------------------

def k1_roofline(prog, k: int, launch_patterns: int, k_ms: float, lane_peak: float, G: int,
                sess) -> dict:
    """Hardware fraction of the dominant kernel (es_k1): LOP3 lane-ops it
    issues per second against the measured LOP3 peak (es_alu_peak).  The
    algorithmic credit (gate-patterns per executed lane-op: LUT-3 mapping x
    cofactor sharing) is reported separately as alg_ops_ratio."""
    from paper_2512_06627_b200 import es

    pipes = es.map_pipes(prog, k)
    iters = launch_patterns / 32 / 2 ** k  # kernel iterations (2^k words each)
    lop3_rate = pipes["lop3"] * iters / (k_ms * 1e-3)
    gate_rate = G * launch_patterns / (k_ms * 1e-3)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("mult16")
        except (OSError, ValueError):
            traffic = None
    return {"bound": "alu", "unit": "lane-LOP3/s", "achieved": lop3_rate, "peak": lane_peak,
            "frac": lop3_rate / lane_peak, "traffic": traffic,
            "kernel": "es_k1", "kernel_ms": k_ms,
            "peak_source": "measured: es_alu_peak (8 independent LOP3 chains per thread, all SMs)",
            "achieved_def": "LOP3 instructions of the kernel body (es.map_pipes) x 32 lanes x "
                            "iterations / kernel time (CUDA events on the launch stream)",
            "lop3_per_iteration": pipes["lop3"], "imad_per_iteration": pipes["imad"],
            "words_per_iteration": 2 ** k, "luts_per_iteration": sess.num_luts,
            "imad_lane_ops_per_s": pipes["imad"] * iters / (k_ms * 1e-3),
            "gate_patterns_per_s": gate_rate,
            "alg_ops_ratio": gate_rate / (lop3_rate * 32),
            "alg_ops_ratio_def": "reference gate-patterns per executed LOP3 lane-op (32 patterns): "
                                 "LUT-3 mapping x cofactor sharing x IMAD offload -- algorithmic "
                                 "credit, not utilisation"}


def k1_two_pipe(prog, k: int, launch_patterns: int, k_ms: float, alu_peak: float, fma_peak: float) -> dict:
    """K1 runs on both integer pipes: LOP3 on the ALU pipe, the x*S+T LUTs,
    their coefficients and the PI masks (IMAD) on the FMA pipe (es_fma_peak:
    the same lane-op peak as the ALU pipe on B200).  The kernel's time is
    bounded by the busier of the two; `frac` here = that pipe's busy time /
    measured time (mult16 k=4: ALU 0.78, FMA 0.47)."""
    from paper_2512_06627_b200 import es

    ptx = es.emit_ptx(prog, 256 if k else 128, k)
    body = ptx[ptx.index(".reg .b32 %esm"):]
    lines = [ln.strip() for ln in body.splitlines()]
    n_lop3 = sum(ln.startswith("lop3.b32") for ln in lines)
    n_fma = sum(ln.startswith(("mad.lo", "mul.lo", "mul.hi")) for ln in lines)
    iters = launch_patterns / 32 / 2 ** k
    alu_s = n_lop3 * iters / alu_peak  # (one thread-iteration issues n lane-ops)
    fma_s = n_fma * iters / fma_peak
    t = k_ms * 1e-3
    return {"alu_peak": alu_peak, "fma_peak": fma_peak, "unit": "lane-ops/s",
            "lop3_per_iteration": n_lop3, "fma_ops_per_iteration": n_fma,
            "alu_frac": alu_s / t, "fma_frac": fma_s / t, "frac": max(alu_s, fma_s) / t,
            "def": "PTX body instructions per iteration (LOP3 -> ALU pipe; mad/mul -> FMA pipe) "
                   "x thread-iterations / each pipe's measured lane-op peak (es_alu_peak, es_fma_peak); frac = the busier "
                   "pipe's busy time / kernel time"}


def ncu_hw(kcof: int):
    """ALU/FMA pipe utilisation of the same kernel from the committed ncu
    summary (the bench itself never runs under a profiler)."""
    name = {4: "r02_k1_cof4_mult16_ncu_full.json"}.get(kcof)
    for cand in filter(None, [name, {4: "r01_k1_cof4_mult16_ncu_full.json"}.get(kcof)]):
        path = os.path.join(ROOT, "profiles", cand)
        if not os.path.exists(path):
            continue
        try:
            d = json.load(open(path))
            pct = lambda k: float(d[k].split()[0])  # noqa: E731
            return {"alu_pipe_pct": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                    "fma_pipe_pct": pct("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                    "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "source": f"profiles/{cand} (ncu --set full, same kernel)"}
        except (OSError, ValueError, KeyError):
            continue
    return None


# --- config 4 (batched cones) ----------------------------------------------

def cones_work(batch, rec) -> tuple[int, int, int]:
    """(gate-patterns, EQ count, NEQ count) of one batched verdict; ``rec`` is
    NativeBatch.run_arrays()'s es_result array."""
    import numpy as np

    tab = batch.table()
    ok = rec["reason"] != -1
    eq = ok & (rec["verdict"] == 0)
    neq = ok & (rec["verdict"] == 1)
    pats = np.where(eq, np.left_shift(np.uint64(1), tab["num_pis"].astype(np.uint64)),
                    rec["patterns_evaluated"])
    work = int((tab["G"].astype(np.float64) * pats.astype(np.float64))[eq | neq].sum())
    return work, int(eq.sum()), int(neq.sum())


def cones_oracle_check(batch, rec) -> dict:
    """Every job of the batched verdict against the CPU oracle's single-worker
    run (verdict, minimum-index witness, patterns_evaluated); raises on any
    mismatch."""
    from oracle import oracle as O

    t = time.perf_counter()
    refs = O.run_packed_batch([batch.packed(i) for i in range(len(batch))])
    codes = {"EXHAUSTED_ZERO": 0, "COUNTEREXAMPLE": 1}
    bad = 0
    for i, g in enumerate(refs):
        if g is None:
            continue
        v = int(rec["verdict"][i])
        w = int(rec["witness_index"][i]) if v == 1 else None
        if (v, w, int(rec["patterns_evaluated"][i])) != (codes[g.verdict], g.witness_index,
                                                         g.patterns_evaluated):
            bad += 1
    if bad:
        raise RuntimeError(f"config 4: {bad} of {len(refs)} jobs differ from the oracle")
    return {"jobs_checked": len(refs), "mismatches": 0, "oracle_s": time.perf_counter() - t}


def k4_issue_model(batch, res) -> dict:
    """Lane-instructions the K4 bodies executed (jobs with engine == JIT in a
    batched run): per job, body instructions (num_luts) x thread-iterations
    (patterns_swept / 32 / 2^k; a thread is one lane).  The skeleton's per-call
    instructions (call, dispatch, fold: ~25) are not counted."""
    import numpy as np

    st = batch.k2_stats()
    k4 = (res["reason"] != -1) & (res["engine"] == 1)
    copies = np.exp2(st["cofactor_pis"].astype(np.float64))
    lane_instrs = res["num_luts"].astype(np.float64) * res["patterns_swept"].astype(np.float64) / (32.0 * copies)
    return {"jobs": int(k4.sum()), "lane_instrs": float(lane_instrs[k4].sum()),
            "body_instrs": int(res["num_luts"][k4].sum())}


def k2_smem_model(batch, res) -> dict:
    """Shared-memory wavefronts the K2 interpreter issues (ncu's
    l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld + _op_st): per warp and
    pass over a job's records, each 16-byte broadcast record load (records +
    the two-step prefetch of the two-lane kernel, 4 records) costs 2
    wavefronts, each slot load or store W (W words x 4 B x 32 threads = W x
    128 B), with the per-program load/store counts of the two-lane schedule
    (accumulator forwarding per lane; a NOP lane loads the zero slot).
    Calibrated against ncu per launch group (profiles/r02_k2l_*)."""
    import numpy as np

    st = batch.k2_stats()
    tr = batch.k2_traffic()
    tab = batch.table()
    ran = (res["reason"] != -1) & (res["engine"] == 2) & (st["num_records"] > 0)
    W = np.maximum(res["regs_per_thread"], 1).astype(np.float64)  # K2 reports its words per thread here
    words = res["patterns_swept"].astype(np.float64) / 32.0  # executed pattern words (all copies)
    copies = np.exp2(st["cofactor_pis"].astype(np.float64))
    iters = words / copies  # interpreter passes over the record list, per thread-word
    warp_iters = iters / (32.0 * W)
    per = 2.0 * (st["num_records"] + 4) + (tr["loads"] + tr["stores"]) * W
    wavefronts = float((warp_iters * per)[ran].sum())
    groups = {}
    for w in (1, 2, 4):
        m = ran & (W == w)
        groups[f"W{w}"] = {"jobs": int(m.sum()),
                           "ld_wavefronts": float((warp_iters * (2.0 * (st["num_records"] + 4)
                                                                 + tr["loads"] * W))[m].sum()),
                           "st_wavefronts": float((warp_iters * tr["stores"] * W)[m].sum())}
    return {"wavefronts": wavefronts, "bytes": wavefronts * 128.0,
            "record_passes": float((iters * st["num_records"])[ran].sum()), "groups": groups}


def measure_cones(steps: int, warmup: int, rank: int = 0, world: int = 1, count: int = 10_000,
                  check: bool = True, cpu_seconds: float = 0.0):
    """Config 4: one batched ES verdict over ~10k candidate-pair cones.
    Device time = the library's CUDA events around the kernel slices (inputs
    resident); e2e = NativeBatch.run wall time (program upload + results)."""
    from paper_2512_06627_b200 import cones, shard

    t = time.perf_counter()
    batches = cones.config4_batches(count)
    sample_ms = 1e3 * (time.perf_counter() - t)  # harness: simulate, pick pairs, extract, compile
    t = time.perf_counter()
    batch = batches[0]
    for b in batches[1:]:
        batch.extend(b)
    batch.prepare()
    prepare_ms = 1e3 * (time.perf_counter() - t)  # K2 programs (cofactor depth, schedule), K4 bodies
    if world > 1:
        batch.select(list(range(rank, len(batch), world)))
    first_ms = None
    for _ in range(warmup):
        t = time.perf_counter()
        res = batch.run_arrays()
        first_ms = first_ms if first_ms is not None else 1e3 * (time.perf_counter() - t)
    dev_ms, wall_ms = [], []
    for _ in range(steps):
        t = time.perf_counter()
        res = batch.run_arrays()
        wall_ms.append(1e3 * (time.perf_counter() - t))
        dev_ms.append(float(res["device_ms"].max()))
    work, eq, neq = cones_work(batch, res)
    smem_bps, _ = shard.smem_peak(0)
    alu_lps, _ = shard.alu_peak(0)
    dev_s = statistics.mean(dev_ms) * 1e-3
    model = k2_smem_model(batch, res)
    k4 = k4_issue_model(batch, res)
    # K4 (the large jobs' straight-line bodies) and K2 (the rest) run
    # concurrently on separate streams; device time is the makespan, so each
    # engine's achieved rate below is a lower bound (its share of the time is
    # in the ncu launch list, profiles/r02_launches_cones.csv)
    roof = {"bound": "issue", "unit": "Tlane-instr/s", "peak": 2.0 * alu_lps / 1e12,
            "peak_source": "measured: 2 x es_alu_peak (LOP3 and IMAD each issue every other cycle "
                           "per scheduler; both pipes together = one instruction per cycle)",
            "achieved": k4["lane_instrs"] / dev_s / 1e12,
            "achieved_def": "K4 body instructions x thread-iterations (jobs of >= 18 PIs) "
                            "/ device makespan",
            "k4": k4}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof_k2 = {"bound": "smem", "unit": "GB/s", "peak": smem_bps / 1e9,
               "peak_source": "measured: es_smem_peak (conflict-free 16-byte shared loads, all SMs)",
               "achieved": model["bytes"] / dev_s / 1e9,
               "achieved_def": "shared-memory wavefronts x 128 B the interpreter issues for the K2 "
                               "jobs (record broadcasts + slot loads/stores after accumulator "
                               "forwarding, per program) / device makespan",
               "wavefronts": model["wavefronts"], "record_passes": model["record_passes"],
               "groups": model["groups"],
               "ncu_check": "profiles/r02_k2l_cones_W*_ncu_full.json: ld/st wavefronts per group"}
    roof_k2["frac"] = roof_k2["achieved"] / roof_k2["peak"]
    roof["k2_part"] = roof_k2
    lt = cones.LAST_TIMING
    out = {"jobs": len(batch), "eq": eq, "neq": neq, "gate_patterns": work, "roofline": roof,
           "device_ms": statistics.mean(dev_ms), "e2e_ms": statistics.mean(wall_ms),
           "host_ms": {"pair_sampling": 1e3 * lt.get("pair_sampling_s", 0.0),
                       "extract_compile": 1e3 * lt.get("extract_compile_s", 0.0),
                       "pairs_extracted": lt.get("pairs_extracted"),
                       "k2_programs_k4_bodies": prepare_ms, "batch_total": sample_ms + prepare_ms,
                       "first_run": first_ms},
           "e2e_with_build_ms": statistics.mean(wall_ms) + prepare_ms
                                + 1e3 * lt.get("extract_compile_s", 0.0) * len(batch)
                                / max(1, lt.get("pairs_extracted") or 1),
           "value": work / dev_s, "e2e_value": work / (statistics.mean(wall_ms) * 1e-3)}
    if check:
        out["oracle_check"] = cones_oracle_check(batch, res)
    if cpu_seconds > 0:
        out["cpu_baseline"] = cones_cpu_baseline(batch, cpu_seconds)
    return out


def measure_cones_eq(steps: int, warmup: int, cpu_seconds: float = 0.0) -> dict:
    """The EQ-heavy config-4 variant: the candidate pairs
    the sweep sends after its 64-word simulation of the configs[2] miter
    alone (cones.sweep_round_batch, sweep.py:313-345) -- mostly EQ cones that
    must be swept completely.  Same measurement as measure_cones, every
    result checked against the oracle."""
    from paper_2512_06627_b200 import cones, shard

    t = time.perf_counter()
    batch = cones.sweep_round_batch()
    build_ms = 1e3 * (time.perf_counter() - t)  # simulate, classes, extract, compile, K2 programs, K4 bodies
    first_ms = None
    for _ in range(warmup):
        t = time.perf_counter()
        res = batch.run_arrays()
        first_ms = first_ms if first_ms is not None else 1e3 * (time.perf_counter() - t)
    dev_ms, wall_ms = [], []
    for _ in range(steps):
        t = time.perf_counter()
        res = batch.run_arrays()
        wall_ms.append(1e3 * (time.perf_counter() - t))
        dev_ms.append(float(res["device_ms"].max()))
    work, eq, neq = cones_work(batch, res)
    dev_s = statistics.mean(dev_ms) * 1e-3
    model = k2_smem_model(batch, res)
    k4 = k4_issue_model(batch, res)
    smem_bps, _ = shard.smem_peak(0)
    alu_lps, _ = shard.alu_peak(0)
    roof = {"bound": "issue", "unit": "Tlane-instr/s", "peak": 2.0 * alu_lps / 1e12,
            "achieved": k4["lane_instrs"] / dev_s / 1e12, "achieved_def": "as for config 4 (k4_issue_model)",
            "k4": k4}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["k2_part"] = {"bound": "smem", "unit": "GB/s", "peak": smem_bps / 1e9,
                       "achieved": model["bytes"] / dev_s / 1e9,
                       "achieved_def": "as for config 4 (k2_smem_model)", "groups": model["groups"]}
    roof["k2_part"]["frac"] = roof["k2_part"]["achieved"] / roof["k2_part"]["peak"]
    out = {"workload": "config 4, EQ-heavy: the 16x16 array-vs-Booth miter's own candidate pairs after a "
                       "64-word simulation (sweep.py:313-345), distinct 14-24-PI cones, one batched launch",
           "jobs": len(batch), "eq": eq, "neq": neq, "gate_patterns": work, "roofline": roof,
           "device_ms": statistics.mean(dev_ms), "e2e_ms": statistics.mean(wall_ms),
           "host_build_ms": build_ms, "first_run_ms": first_ms,
           "e2e_with_build_ms": statistics.mean(wall_ms) + build_ms,
           "value": work / dev_s, "e2e_value": work / (statistics.mean(wall_ms) * 1e-3),
           "oracle_check": cones_oracle_check(batch, res)}
    if cpu_seconds > 0:
        out["cpu_baseline"] = cones_cpu_baseline(batch, cpu_seconds)
    return out


def _ref_cone_worker(args):
    """One process of the N-process reference harness: es_check(workers=1) on
    its share of the cones (the reference's own call, es.py:342)."""
    items, seconds = args
    ref = reference_pkg()
    from paper_2512_06627_b200.xag import Gate, GateKind, Lit, Xag

    work, n, t0 = 0, 0, time.perf_counter()
    for (npis, kind, in0, in1, out) in items:
        x = Xag(npis, tuple(Gate(GateKind(int(k)), Lit.unpack(int(a)), Lit.unpack(int(b)))
                            for k, a, b in zip(kind, in0, in1)), (Lit.unpack(int(out)),))
        rx = to_ref(x, ref)
        p = ref.es.compile_program(rx)
        r = ref.es.run_exhaustive(p, workers=1)
        work += _ref_G(p) * r.patterns_evaluated
        n += 1
        if time.perf_counter() - t0 > seconds:
            break
    return work, n, time.perf_counter() - t0


def cones_cpu_baseline(batch, seconds: float) -> dict:
    """the reference's per-cone ES (compile +
    run_exhaustive, workers=1) in a loop on one core, and the same harness on
    every host core (one process per core, cones dealt round-robin)."""
    import multiprocessing as mp

    ref = reference_pkg()
    items = [batch.packed(i) for i in range(len(batch))]
    if ref is None:
        return {"unavailable": "baseline/_ref missing"}
    _ref_cone_worker((items[:2], 1.0))  # numba JIT outside the timing
    w1, n1, s1 = _ref_cone_worker((items, seconds / 2))
    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        parts = pool.map(_ref_cone_worker, [(items[c::cores], seconds / 2) for c in range(cores)])
    wn = sum(p[0] for p in parts)
    nn = sum(p[1] for p in parts)
    sn = max(p[2] for p in parts)
    best_all = wn / sn
    return {"value": max(w1 / s1, best_all), "unit": UNIT, "cores": cores if best_all > w1 / s1 else 1,
            "kind": "reference",
            "sample": f"cecprove es compile_program + run_exhaustive(workers=1) per cone (baseline/_ref): "
                      f"1 core {n1} cones in {s1:.1f}s; {cores} processes {nn} cones in {sn:.1f}s",
            "per_core": {"value": w1 / s1, "cones": n1, "seconds": s1},
            f"processes_{cores}": {"value": best_all, "cones": nn, "seconds": sn}}


# --- other measurements ----------------------------------------------------

def measure_random_sim(local: int, words: int = 1 << 16, cpu: bool = True) -> dict:
    """K3 random simulation of the mult16 miter (every node
    row written to HBM: 8 bytes per node per 64-pattern word), drive and
    output resident; plus the sweep's 64-word PE-class discovery end to end."""
    import numpy as np
    import torch

    from paper_2512_06627_b200 import sim

    x, _ = build_workload("mult16")
    nn = 1 + x.num_pis + len(x.gates)
    pw = sim.random_pi_words(x.num_pis, words, 1)
    d_pi = torch.from_numpy(pw.view(np.int64)).to(f"cuda:{local}")
    d_out = torch.empty((nn, words), dtype=torch.int64, device=f"cuda:{local}")
    ds = sim.DeviceSim(x)
    st = torch.cuda.current_stream(local)
    for _ in range(3):
        ds.run(d_pi.data_ptr(), words, d_out.data_ptr(), st.cuda_stream)
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ds.run(d_pi.data_ptr(), words, d_out.data_ptr(), st.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ds.close()
    peak = None
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        pass
    written = nn * words * 8
    gbs = written / (ms * 1e-3) / 1e9
    sim.pe_classes(x, 64, 0, device=local)  # warm
    walls = []
    for s in range(5):
        t = time.perf_counter()
        n_cls = len(sim.pe_classes(x, 64, s, device=local))
        walls.append(1e3 * (time.perf_counter() - t))
    out = {"workload": f"random simulation of the 16x16 array-vs-Booth miter, {words} 64-bit words "
                       "per node (sim.py:21-38), device-resident drive and node matrix",
           "device_ms": ms, "gate_patterns_per_s": len(x.gates) * words * 64 / (ms * 1e-3),
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                        "frac": None if peak is None else gbs / peak,
                        "algorithmic_bytes": written,
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"},
           "pe_classes_64_words_e2e_ms": statistics.median(walls), "pe_classes": n_cls}
    if cpu:  # the reference algorithm restated in numpy (oracle/), same drive
        from oracle import oracle as O
        pw64 = sim.random_pi_words(x.num_pis, 64, 0)
        t = time.perf_counter()
        O.pe_classes(O.simulate(x, pw64))
        out["cpu_pe_classes_64_words_ms"] = 1e3 * (time.perf_counter() - t)
        small = sim.random_pi_words(x.num_pis, 4096, 1)
        t = time.perf_counter()
        O.simulate(x, small)
        out["cpu_simulate_4096_words_ms"] = 1e3 * (time.perf_counter() - t)
    return out


def measure_sweep(local: int) -> dict:
    """the whole sweep with the ES engine (sweep.py:292-409)
    on the config-2/3 multiplier miters -- K3 simulation and classes, C++
    extraction, batched K2 / parallel-JIT K1 pair checks, final obligation.
    Cold = first sweep of the miter in this process (JIT included); warm =
    the best of three repeats."""
    from paper_2512_06627_b200 import miter as M
    from paper_2512_06627_b200.sweep import SweepConfig, sweep

    out = {}
    for name, (w, a, b) in {"mult12": (12, "array", "wallace"), "mult16": (16, "array", "booth")}.items():
        x = M.gen_multiplier_miter(w, a, b)
        t = time.perf_counter()
        r = sweep(x, SweepConfig(device=local))
        cold = 1e3 * (time.perf_counter() - t)
        # repeat sweeps: the second one still pays the policy's tier-up (deeper
        # cofactor variants mapped and built because the sub-miters re-run);
        # warm = the best of three repeats (kernels built and tiered up)
        reps = []
        for _ in range(3):
            t = time.perf_counter()
            sweep(x, SweepConfig(device=local))
            reps.append(1e3 * (time.perf_counter() - t))
        warm = min(reps)
        out[name] = {"verdict": r.verdict, "cold_ms": cold, "warm_ms": warm, "repeat_ms": reps,
                     "pairs_checked": r.stats["engine_calls"], "merges": r.stats["merges"],
                     "reference_sweep_s_1_thread_build_container": {"mult12": 6.78, "mult16": 376.89}[name]}
    return out


def measure_other_configs(local: int, cofactor="throughput", cpu_seconds: float = 0.0) -> dict:
    """Short warm measurements of the other BASELINE.json configs on 1 GPU,
    each with the reference's CPU ES beside it."""
    from paper_2512_06627_b200 import es

    out = {}
    for name in ("adder8", "mult12", "mult16_neq"):
        x, desc = build_workload(name)
        # cold: the first call in the process under the default latency policy
        # (what a one-off es_check costs, JIT included; cubin cache off in run_b200)
        t = time.perf_counter()
        p = es.compile_program(x)
        cold = es.run_exhaustive(p, engine="auto", device=local)
        cold_ms = 1e3 * (time.perf_counter() - t)
        es.run_exhaustive(p, engine="auto", device=local, cofactor=cofactor)  # warm-up (JIT of the mode)
        devs, walls = [], []
        for _ in range(10):
            t = time.perf_counter()
            r = es.es_check(_Sub(x), engine="auto", device=local, cofactor=cofactor)
            walls.append(1e3 * (time.perf_counter() - t))
            devs.append(r.stats["device_ms"])
        pats = (1 << x.num_pis) if r.verdict == "EQUIVALENT" else r.stats["patterns"]
        dev = statistics.median(devs)
        row = {"workload": desc, "verdict": r.verdict,
               "witness_index": None if r.witness is None else
               sum(b << i for i, b in enumerate(r.witness)),
               "engine": r.stats["engine"], "device_ms": dev,
               "e2e_ms": statistics.median(walls), "cold_ms": cold_ms,
               "cold_engine": cold.stats["engine"], "cold_jit_ms": cold.stats["jit_ms"],
               "gate_patterns_per_s": p.num_gates * pats / (dev * 1e-3),
               "patterns_swept": r.stats["patterns_swept"], "phases": r.stats["phases"],
               "phase2_copies": r.stats["phase2_copies"],
               "phase2_cofactor_pis": r.stats["phase2_cofactor_pis"]}
        if cpu_seconds > 0:
            cb = cpu_baseline(x, cpu_seconds)
            row["cpu_baseline"] = cb
            if "time_to_verdict_s" in cb:
                row["speedup_time_to_verdict_vs_cpu"] = cb["time_to_verdict_s"] * 1e3 / row["e2e_ms"]
            else:  # rate-based: the CPU's time to the same verdict at its measured rate
                row["cpu_time_to_verdict_est_s"] = p.num_gates * pats / cb["value"]
        out[name] = row
    eq = out.get("mult16_neq")
    return out


def disk_cache_ttv(config: str, cofactor) -> dict:
    """Cold time-to-verdict in a fresh process with the on-disk cubin cache
    (es_jit.cpp) populated by a previous process: compile + map + load + sweep,
    no ptxas.  Two child processes on a private cache directory."""
    code = ("import sys, time, json; sys.path.insert(0, %r)\n"
            "from bench import build_workload\n"
            "from paper_2512_06627_b200 import es\n"
            "x, _ = build_workload(%r)\n"
            "from paper_2512_06627_b200 import miter as M\n"
            "es.run_exhaustive(es.compile_program(M.gen_adder_miter(4)), engine='interp')  # CUDA context\n"
            "t = time.perf_counter(); r = es.run_exhaustive(es.compile_program(x), engine='jit', cofactor=%r)\n"
            "print(json.dumps({'ms': 1e3 * (time.perf_counter() - t), 'jit_ms': r.stats['jit_ms']}))\n"
            % (ROOT, config, cofactor))
    out = {}
    with tempfile.TemporaryDirectory() as d:
        env = dict(os.environ, ES_JIT_CACHE="1", ES_JIT_CACHE_DIR=d)
        for tag in ("populate", "warm_disk"):
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                               timeout=600)
            if r.returncode != 0:
                return {"error": r.stderr[-300:]}
            out[tag] = json.loads(r.stdout.strip().splitlines()[-1])
    return {"cold_ms_disk_cache": out["warm_disk"]["ms"], "jit_ms_disk_cache": out["warm_disk"]["jit_ms"],
            "cold_ms_first_process": out["populate"]["ms"]}


# --- the reference arm -----------------------------------------------------

def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    ref = reference_pkg()
    # each step a bounded sample so the whole run ends within a few minutes
    per_step = max(0.3, min(5.0, 150.0 / max(1, args.steps + args.warmup)))
    base = {"metric": METRIC, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64 (bit-parallel words)", "data": "synthetic",
            "impl": "reference"}
    if args.config == "cones":
        from paper_2512_06627_b200 import cones
        batch = cones.config4_batch(10_000)
        items = [batch.packed(i) for i in range(len(batch))]
        _ref_cone_worker((items[:2], 1.0))
        work = 0
        el = 0.0
        for s in range(args.warmup + args.steps):
            w, n, dt = _ref_cone_worker((items[(s * 97) % len(items):], per_step))
            if s >= args.warmup:
                work, el = work + w, el + dt
        value = work / el
        line = dict(base, value=value, ms_per_step=1e3 * el / args.steps,
                    config={"workload": "config 4: ~10k candidate-pair cones (14-24 PIs) of 16x16 "
                                        "multiplier miters", "step": f"{per_step:.2f}s of per-cone ES"},
                    cpu_baseline={"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                                  "sample": f"cecprove compile_program + run_exhaustive(workers=1) per "
                                            f"cone, {per_step:.2f}s per step"},
                    e2e={"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return
    x, desc = build_workload(args.config)
    if ref is None:  # the oracle's C restatement (kind "port")
        from oracle import oracle as O
        p = O.compile_program(x)
        G = p.num_gate_instrs
        per_batch = 1 << min(x.num_pis, 14)
        total_batches = 1 << max(x.num_pis - 14, 0)
        probe = min(total_batches, 64 * cores)
        O.min_witness(p, threads=cores, max_batches=probe)
        t = time.perf_counter()
        O.min_witness(p, threads=cores, max_batches=probe)
        dt = max(time.perf_counter() - t, 1e-6)
        nb = int(min(total_batches, max(probe, probe * per_step / dt)))
        for _ in range(args.warmup):
            O.min_witness(p, threads=cores, max_batches=nb)
        t = time.perf_counter()
        done = sum(O.min_witness(p, threads=cores, max_batches=nb)[2] for _ in range(args.steps))
        el = time.perf_counter() - t
        value = G * done * per_batch / el
        kind, sample = "port", f"{nb} batches x 2^{min(x.num_pis, 14)} patterns per step (oracle C port)"
    else:
        p = ref.es.compile_program(to_ref(x, ref))
        G = _ref_G(p)
        ref.es.run_exhaustive(p, workers=cores, budget=0.05)  # numba JIT
        for _ in range(args.warmup):
            ref.es.run_exhaustive(p, workers=cores, budget=per_step)
        pats, el = 0, 0.0
        verdicts = set()
        for _ in range(args.steps):
            t = time.perf_counter()
            r = ref.es.run_exhaustive(p, workers=cores, budget=per_step)
            el += time.perf_counter() - t
            pats += r.patterns_evaluated
            verdicts.add(r.verdict)
        value = G * pats / el
        kind = "reference"
        sample = (f"cecprove.es.run_exhaustive(compile_program(x), workers={cores}, budget="
                  f"{per_step:.2f}s) per step (baseline/_ref, numba); verdicts {sorted(verdicts)}")
    line = dict(base, value=value, ms_per_step=1e3 * el / args.steps,
                config={"workload": desc, "num_pis": x.num_pis, "G": G,
                        "step": f"bounded sample: {per_step:.2f}s of the same sweep"},
                cpu_baseline={"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
                e2e={"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    print(json.dumps(line), flush=True)


# --- the B200 arm ----------------------------------------------------------

def run_b200(args) -> None:
    import torch

    # cold numbers below are true cold: no on-disk cubin cache in this process
    os.environ["ES_JIT_CACHE"] = "0"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and world != args.gpus:
        raise SystemExit(f"bench: torchrun WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.cofactor.isdigit():
        args.cofactor = int(args.cofactor)
    if world > 1:
        run_ranks(args, world)
        return
    from paper_2512_06627_b200 import es

    visible = es.device_count()
    if visible < args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but only {visible} CUDA device(s) visible")
    if args.config == "cones":
        run_cones(args)
        return
    run_local(args, list(range(args.gpus)))


def run_local(args, devs: list[int]) -> None:
    """N GPUs driven by ONE es_run call (es_run_opts.devices), or 1 GPU."""
    import torch

    from paper_2512_06627_b200 import es, shard

    N = len(devs)
    devices = devs if N > 1 else None
    x, desc = build_workload(args.config)
    sm = _Sub(x)
    P = x.num_pis
    for d in devs:
        torch.cuda.set_device(d)
        shard.alu_peak(d)  # CUDA context + module load outside the cold measurement
    torch.cuda.set_device(devs[0])
    # cold time-to-verdict: compile + map + JIT + sweep, first call in process,
    # in the default latency mode (cofactor="auto") and in this run's mode
    t = time.perf_counter()
    prog = es.compile_program(x)
    cold = es.run_exhaustive(prog, engine="jit", cofactor="auto", devices=devices)
    cold_ms = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter()
    cold_t = es.run_exhaustive(es.compile_program(x), engine="jit", cofactor=args.cofactor, devices=devices)
    cold_t_ms = 1e3 * (time.perf_counter() - t)
    G = prog.num_gates
    if (cold_t.verdict, cold_t.witness_index) != (cold.verdict, cold.witness_index):
        raise RuntimeError("cofactor modes disagree")
    expected = (cold.verdict, cold.witness_index)
    flush = [torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{d}") for d in devs]

    def step():
        r = es.run_exhaustive(prog, engine="jit", cofactor=args.cofactor, devices=devices)
        if (r.verdict, r.witness_index) != expected:
            raise RuntimeError(f"verdict drift: {r.verdict} {r.witness_index} vs {expected}")
        return r

    def sync():
        for d in devs:
            torch.cuda.synchronize(d)

    for _ in range(args.warmup):
        step()
        for f in flush:
            f.zero_()
    sync()
    # timed region: K verdicts; device time of each = the library's CUDA events
    # around its launch slices (max over the GPUs); L2 flushed between verdicts
    dev_ms, host_ms = [], []
    with ClockSampler(devs) as clk:
        for _ in range(args.steps):
            t = time.perf_counter()
            r = step()
            host_ms.append(1e3 * (time.perf_counter() - t))
            dev_ms.append(r.stats["device_ms"])
            for f in flush:
                f.zero_()
            sync()
    total_s = sum(dev_ms) * 1e-3
    patterns_per_step = (1 << P) if r.witness_index is None else min(1 << P, r.patterns_evaluated)
    value = G * patterns_per_step * args.steps / total_s

    # dominant kernel (es_k1) alone on GPU 0: one launch over the whole space
    sess = shard.session_for(prog, devs[0], args.cofactor)
    dev = torch.device(f"cuda:{devs[0]}")
    best = torch.empty(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(max(args.steps, 5))]
    for a, b in kev:
        best.fill_(1 << P)
        flush[0].zero_()
        a.record()
        sess.launch(stream, best.data_ptr(), 0, sess.n_chunks, 0, 1)
        b.record()
    torch.cuda.synchronize(dev)
    k_ms = statistics.mean(a.elapsed_time(b) for a, b in kev)
    launch_patterns = sess.n_chunks * sess.patterns_per_chunk
    if r.witness_index is not None:
        launch_patterns = min(launch_patterns, r.stats["patterns_swept"])
    lane_peak, _ = shard.alu_peak(devs[0])
    kcof = cold_t.stats.get("cofactor_pis", 0)
    roof = k1_roofline(prog, kcof, launch_patterns, k_ms, lane_peak, G, sess)
    roof["hardware"] = ncu_hw(kcof) if args.config == "mult16" else None
    roof["two_pipe"] = k1_two_pipe(prog, kcof, launch_patterns, k_ms, lane_peak, shard.fma_peak(devs[0])[0])

    # e2e through the public API: host circuit in, host verdict out
    for _ in range(max(1, args.warmup)):
        es.es_check(sm, engine="jit", cofactor=args.cofactor, devices=devices)
    e_ms, launches = [], []
    for _ in range(args.steps):
        t = time.perf_counter()
        res = es.es_check(sm, engine="jit", cofactor=args.cofactor, devices=devices)
        e_ms.append(1e3 * (time.perf_counter() - t))
        launches.append(res.stats["launches"])
    e2e_value = G * patterns_per_step * args.steps / (sum(e_ms) * 1e-3)

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(x, args.cpu_seconds)
    mode_desc = (f"{N} GPUs in one es_run call (es_run_opts.devices): chunks dealt round-robin, one "
                 "host thread per GPU, one minimum word in GPU 0's HBM shared as NVLink peer memory "
                 "(kernel atomicMin + skip rule), no collective" if N > 1 else "1 GPU, es_run")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_s * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u32 (bit-parallel LOP3 words)", "data": "synthetic",
        "config": {"workload": desc, "num_pis": P, "G": G, "patterns_per_step": patterns_per_step,
                   "verdict": r.verdict, "witness_index": r.witness_index,
                   "parallelism": mode_desc,
                   "l2": "flushed between steps (256 MiB write per GPU, outside the step's device "
                         "time); the kernel reads no HBM inputs",
                   "cofactor_pis": kcof, "words_per_iteration": 2 ** kcof,
                   "luts_per_iteration": sess.num_luts, "luts_per_word": sess.num_luts / 2 ** kcof,
                   "regs_per_thread": sess.regs_per_thread, "phases": r.stats["phases"],
                   "patterns_swept": r.stats["patterns_swept"],
                   "host_ms_per_step": statistics.mean(host_ms)},
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                "d2h_bytes_per_step": 20 * int(statistics.mean(launches)),
                "path": "es.es_check(sub-miter) -> compile_program -> C ABI es_run (host circuit in, "
                        "host verdict out; JIT module cached by program hash)",
                "ms_per_step": statistics.mean(e_ms)},
        "time_to_verdict": {"cold_ms": cold_ms, "jit_ms": cold.stats.get("jit_ms"),
                            "host_compile_ms": cold.stats.get("compile_ms"),
                            "device_ms": cold.stats.get("device_ms"),
                            "mode": f"cofactor=auto (latency), k={cold.stats.get('cofactor_pis')}",
                            f"cold_ms_{args.cofactor}": cold_t_ms,
                            f"jit_ms_{args.cofactor}": cold_t.stats.get("jit_ms"),
                            f"device_ms_{args.cofactor}": cold_t.stats.get("device_ms"),
                            "warm_device_ms": total_s * 1e3 / args.steps,
                            "note": "cold = first call in a process, JIT included, on-disk cubin "
                                    "cache off"},
        "gpu_launches": int(sum(launches)),
        "clocks": clk.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["cpu_baseline"]["detail"] = {k: v for k, v in cpu.items()
                                          if k not in ("value", "unit", "cores", "kind", "sample")}
    if N == 1 and not args.no_extras:
        for mode in ("auto", args.cofactor):
            line["time_to_verdict"][f"disk_cache_{mode}"] = disk_cache_ttv(args.config, mode)
        # the GPU idled (down-clocked) during the child processes: bring the
        # clocks back up before the short extra measurements
        t_end = time.perf_counter() + 0.5
        while time.perf_counter() < t_end:
            sess.launch(stream, best.data_ptr(), 0, sess.n_chunks, 0, 1)
            torch.cuda.synchronize(dev)
        cs = 0.0 if args.no_cpu_baseline else args.extra_cpu_seconds
        extras = measure_other_configs(devs[0], args.cofactor, cs)
        extras["random_sim"] = measure_random_sim(devs[0], cpu=not args.no_cpu_baseline)
        extras["sweep_es"] = measure_sweep(devs[0])
        extras["cones"] = {"workload": "config 4: ~10k candidate-pair cones (14-24 PIs) of "
                                       "16x16 multiplier miters, one batched launch",
                           **measure_cones(5, 2, cpu_seconds=cs)}
        extras["cones_eq"] = measure_cones_eq(5, 2, cpu_seconds=cs)
        line["other_configs"] = extras
    print(json.dumps(line), flush=True)


def run_ranks(args, world: int) -> None:
    """torchrun: one process per GPU, each sweeping its residue class of
    chunks; one shared minimum word per verdict (CUDA IPC into rank 0's HBM,
    NVLink peer memory) closed by a device-side barrier, verdicts queued
    back to back (p2p), or the NCCL MIN all-reduce fallback (--collective nccl)."""
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.backend == "nccl":
        if torch.cuda.device_count() < world:
            raise SystemExit(f"bench: {world} ranks but {torch.cuda.device_count()} GPUs visible")
    else:  # --backend gloo lets several ranks share one GPU (tests only)
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(args.backend)
    from paper_2512_06627_b200 import es, shard

    if args.config == "cones":
        run_cones(args, rank, world, local, dev)
        return
    x, desc = build_workload(args.config)
    P = x.num_pis
    prog = es.compile_program(x)
    G = prog.num_gates
    expected = es.run_exhaustive(prog, engine="jit", cofactor=args.cofactor, device=local)
    sess = shard.session_for(prog, local, args.cofactor)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    collective = args.collective
    peer = None
    if collective == "p2p":
        try:
            peer = shard.PeerBest(None, local)
        except Exception as exc:  # no IPC / peer access: fall back to NCCL MIN
            print(f"[bench] peer word unavailable ({exc}); using NCCL all-reduce", file=sys.stderr)
            collective = "nccl"
    S = args.slices or 4
    best = torch.empty(1, dtype=torch.int64, device=dev)
    n = args.warmup + args.steps
    outs = torch.empty(n, dtype=torch.int64, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]

    def verdict(i: int):
        if peer is not None:  # queued: no host synchronisation
            shard.sweep_peer_async(prog, peer, outs[i].data_ptr(), local, args.cofactor)
        else:
            r = shard.sweep_sharded(prog, None, local, slices=S, best=best, cofactor=args.cofactor)
            outs[i].fill_(r.witness_index if r.witness_index is not None else (1 << 64) - 1 - (1 << 63) * 2)

    for i in range(args.warmup):
        verdict(i)
        flush.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            evs[i][0].record()
            verdict(args.warmup + i)
            evs[i][1].record()
            flush.zero_()
        torch.cuda.synchronize()
    dist.barrier()
    words = [int(v) & 0xFFFFFFFFFFFFFFFF for v in outs.tolist()]
    want = expected.witness_index
    for w in words:
        got = w if w < (1 << P) else None
        if got != want:
            raise RuntimeError(f"rank {rank}: verdict drift {got} vs {want}")
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    dist.all_reduce(total, op=dist.ReduceOp.MAX)
    total_s = float(total.item()) * 1e-3
    patterns_per_step = (1 << P) if want is None else min(1 << P, expected.patterns_evaluated)
    value = G * patterns_per_step * args.steps / total_s
    # e2e: es_check through the sharded API, host circuit in, host verdict out
    sm = _Sub(x)
    e_ms = []
    for i in range(max(1, args.warmup) + args.steps):
        dist.barrier()
        t = time.perf_counter()
        if peer is not None:
            shard.es_check_peer(sm, peer, None, local, cofactor=args.cofactor)
        else:
            shard.es_check_sharded(sm, None, local, slices=S, cofactor=args.cofactor)
        if i >= max(1, args.warmup):
            e_ms.append(1e3 * (time.perf_counter() - t))
    e_total = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
    dist.all_reduce(e_total, op=dist.ReduceOp.MAX)
    e2e_value = G * patterns_per_step * args.steps / (float(e_total.item()) * 1e-3)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_s * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32 (bit-parallel LOP3 words)", "data": "synthetic",
            "config": {"workload": desc, "num_pis": P, "G": G, "patterns_per_step": patterns_per_step,
                       "verdict": expected.verdict, "witness_index": want,
                       "parallelism": (f"torchrun x{world}: pattern-space shards, one minimum word in "
                                       "rank 0's HBM mapped into every rank (CUDA IPC / NVLink peer "
                                       "memory), kernel atomicMin + skip rule, device-side verdict "
                                       "barrier (es_peer_arrive_wait), verdicts queued back to back"
                                       if collective == "p2p" else
                                       f"torchrun x{world}: pattern-space shards, NCCL MIN all-reduce "
                                       f"after each of {S} launch slice(s)"),
                       "l2": "flushed between steps (256 MiB write, outside the step events)",
                       "cofactor_pis": expected.stats["cofactor_pis"],
                       "luts_per_iteration": sess.num_luts},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8, "d2h_bytes_per_step": 8,
                    "path": "shard.es_check_peer -> compile_program -> session launch + device barrier"
                            if collective == "p2p" else "shard.es_check_sharded",
                    "ms_per_step": float(e_total.item()) / args.steps},
            "gpu_launches": args.steps * world * (3 if collective == "p2p" else S),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    dist.destroy_process_group()


def run_cones(args, rank: int = 0, world: int = 1, local: int = 0, dev=None) -> None:
    """Config 4 as the headline workload (--config cones)."""
    import torch
    import torch.distributed as dist

    with ClockSampler(local) as clk:
        m = measure_cones(args.steps, args.warmup, rank, world, check=True,
                          cpu_seconds=0.0 if args.no_cpu_baseline or rank else args.extra_cpu_seconds)
    if world > 1:
        t = torch.tensor([m["device_ms"], m["e2e_ms"]], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        w = torch.tensor([m["gate_patterns"]], dtype=torch.float64, device=dev)
        dist.all_reduce(w)
        work = float(w.item())
        dev_ms, e2e_ms = float(t[0]), float(t[1])
    else:
        work, dev_ms, e2e_ms = m["gate_patterns"], m["device_ms"], m["e2e_ms"]
    if rank == 0:
        line = {"metric": METRIC, "value": work / (dev_ms * 1e-3), "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": dev_ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u32 (bit-parallel words)", "data": "synthetic",
                "config": {"workload": "config 4: ~10k candidate-pair cones (14-24 PIs) of 16x16 "
                                       "multiplier miters, batched K2 launch",
                           "jobs_rank0": m["jobs"], "eq_rank0": m["eq"], "neq_rank0": m["neq"],
                           "host_ms": m["host_ms"],
                           "parallelism": f"jobs dealt round-robin over {world} GPU(s)"},
                "roofline": m["roofline"], "oracle_check": m.get("oracle_check"),
                "e2e": {"value": work / (e2e_ms * 1e-3), "unit": UNIT,
                        "ms_per_step": e2e_ms, "h2d_bytes_per_step": None,
                        "d2h_bytes_per_step": None},
                "gpu_launches": args.steps * world * 3, "clocks": clk.summary()}
        if "cpu_baseline" in m:
            line["cpu_baseline"] = m["cpu_baseline"]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--config", default="mult16")
    ap.add_argument("--slices", type=int, default=0)
    ap.add_argument("--cofactor", default="throughput",
                    help="K1 cofactor mode: throughput (default), auto, none, or 1..5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--extra-cpu-seconds", type=float, default=6.0,
                    help="CPU baseline budget of each other_configs entry")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--backend", default="nccl", help="torch.distributed backend under torchrun")
    ap.add_argument("--collective", choices=("p2p", "nccl"), default="p2p",
                    help="torchrun exchange: shared peer word (p2p) or NCCL MIN per slice")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
