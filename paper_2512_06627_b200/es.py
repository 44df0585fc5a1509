"""Exact-simulation engine on B200: the drop-in for cecprove/es.py.

Same public surface and contract as the reference module (es.py:25-365,
SPEC.md:305-369): ``compile_program``, ``run_exhaustive``, ``es_check``,
``Instr``, ``InstrProgram``, ``EsResult``, ``TooManyInputs``, the op codes and
verdict strings.  ``es_check(sm, workers, budget, cancel)`` can replace the
reference's in ``sched.dispatch`` (sched.py:236-238) and
``sweep._check_submiter`` (sweep.py:240-243) unchanged.

Differences that are deliberate and documented:
  * the sweep runs on a GPU (libes_b200.so); ``workers`` keeps its meaning for
    argument validation (>= 1, es.py:260-261) but parallelism is the GPU's;
  * the counterexample is always the minimum-index failing pattern -- the
    reference's ``workers=1`` witness -- for any ``workers``;
  * ``patterns_evaluated`` uses the reference's workers=1 accounting
    (batches of 2^min(n,14) patterns up to and including the hit).
There is no CPU fallback: without the native library or a GPU, calls raise.
"""

from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, Iterable, Sequence

import numpy as np

from . import _native as N
from .miter import evaluate
from .verdict import COUNTEREXAMPLE, EQUIVALENT, UNKNOWN, CheckResult
from .xag import packed_gates

MAX_ES_PIS = 40

OP_LOAD_PI = 0
OP_AND = 1
OP_XOR = 2
OP_OUTPUT = 3

_OP_NAMES = {OP_LOAD_PI: "load", OP_AND: "and", OP_XOR: "xor", OP_OUTPUT: "out"}

EXHAUSTED_ZERO = "EXHAUSTED_ZERO"
ES_COUNTEREXAMPLE = "COUNTEREXAMPLE"
BUDGET_EXCEEDED = "BUDGET_EXCEEDED"
_VERDICTS = (EXHAUSTED_ZERO, ES_COUNTEREXAMPLE, BUDGET_EXCEEDED)


class TooManyInputs(ValueError):
    pass


@dataclass(frozen=True)
class Instr:
    """One register operation (es.py:43-63); src -1 is the constant-0 rail."""

    op: int
    dst: int = 0
    src0: int = -1
    neg0: bool = False
    src1: int = -1
    neg1: bool = False
    pi: int = 0

    def render(self) -> str:
        if self.op == OP_LOAD_PI:
            return f"r{self.dst} = load pi{self.pi}"
        a = f"{'~' if self.neg0 else ''}r{self.src0}" if self.src0 >= 0 else (
            "const1" if self.neg0 else "const0")
        if self.op == OP_OUTPUT:
            return f"out {a}"
        b = f"{'~' if self.neg1 else ''}r{self.src1}"
        return f"r{self.dst} = {a} {_OP_NAMES[self.op]} {b}"


class InstrProgram:
    """The reference InstrProgram (es.py:66-73) backed by the SoA arrays the
    C ABI takes (es.py:_encode, :232-249).  ``instrs`` materialises lazily."""

    __slots__ = ("op", "dst", "src0", "neg0", "src1", "neg1", "pi", "num_registers",
                 "num_pis", "_instrs", "_struct")

    def __init__(self, op, dst, src0, neg0, src1, neg1, pi, num_registers: int, num_pis: int):
        self.op = np.ascontiguousarray(op, dtype=np.int8)
        self.dst = np.ascontiguousarray(dst, dtype=np.int32)
        self.src0 = np.ascontiguousarray(src0, dtype=np.int32)
        self.neg0 = np.ascontiguousarray(neg0, dtype=np.uint8)
        self.src1 = np.ascontiguousarray(src1, dtype=np.int32)
        self.neg1 = np.ascontiguousarray(neg1, dtype=np.uint8)
        self.pi = np.ascontiguousarray(pi, dtype=np.int32)
        self.num_registers = int(num_registers)
        self.num_pis = int(num_pis)
        self._instrs = None
        self._struct = None

    @classmethod
    def from_instrs(cls, instrs: Sequence, num_registers: int, num_pis: int) -> "InstrProgram":
        """Adopt any Instr sequence (this module's or the reference's)."""
        rows = [(i.op, i.dst, i.src0, int(i.neg0), i.src1, int(i.neg1), i.pi) for i in instrs]
        a = np.array(rows, dtype=np.int64).reshape(-1, 7)
        return cls(a[:, 0], a[:, 1], a[:, 2], a[:, 3], a[:, 4], a[:, 5], a[:, 6],
                   num_registers, num_pis)

    @property
    def instrs(self) -> tuple[Instr, ...]:
        if self._instrs is None:
            self._instrs = tuple(
                Instr(int(o), int(d), int(a), bool(na), int(b), bool(nb), int(p))
                for o, d, a, na, b, nb, p in zip(self.op, self.dst, self.src0, self.neg0,
                                                 self.src1, self.neg1, self.pi))
        return self._instrs

    @property
    def num_gates(self) -> int:
        """G: AND+XOR instructions -- the work unit of gate-patterns/s."""
        return int(np.count_nonzero((self.op == OP_AND) | (self.op == OP_XOR)))

    def rows(self) -> list[list[int]]:
        return [[int(v) for v in r] for r in zip(self.op, self.dst, self.src0, self.neg0,
                                                  self.src1, self.neg1, self.pi)]

    def dump(self) -> str:
        return "\n".join(i.render() for i in self.instrs)

    def __len__(self) -> int:
        return int(self.op.shape[0])

    def __eq__(self, other) -> bool:
        if not isinstance(other, InstrProgram):
            return NotImplemented
        return (self.num_registers == other.num_registers and self.num_pis == other.num_pis
                and self.rows() == other.rows())

    def __repr__(self) -> str:
        return (f"InstrProgram(<{len(self)} instrs>, num_registers={self.num_registers}, "
                f"num_pis={self.num_pis})")

    def as_struct(self) -> N.EsProg:
        if self._struct is None:
            s = N.EsProg()
            s.num_instrs = len(self)
            s.num_registers = self.num_registers
            s.num_pis = self.num_pis
            for f in ("op", "dst", "src0", "neg0", "src1", "neg1", "pi"):
                setattr(s, f, getattr(self, f).ctypes.data)
            self._struct = s
        return self._struct


def as_program(p) -> InstrProgram:
    if isinstance(p, InstrProgram):
        return p
    return InstrProgram.from_instrs(p.instrs, p.num_registers, p.num_pis)


@dataclass
class EsResult:
    verdict: str  # EXHAUSTED_ZERO | COUNTEREXAMPLE | BUDGET_EXCEEDED
    witness: tuple[int, ...] | None = None
    patterns_evaluated: int = 0
    witness_index: int | None = None
    stats: dict = field(default_factory=dict)

    def __post_init__(self) -> None:
        if (self.witness is not None) != (self.verdict == ES_COUNTEREXAMPLE):
            raise ValueError("witness present iff verdict is COUNTEREXAMPLE")


def compile_program(xag) -> InstrProgram:
    """Reference schedule (es.py:87-163), computed by the native compiler."""
    if len(xag.outputs) != 1:
        raise ValueError(f"expected single output, found {len(xag.outputs)}")
    n, g = xag.num_pis, len(xag.gates)
    if n > MAX_ES_PIS:
        raise TooManyInputs(f"{n} PIs exceeds the {MAX_ES_PIS} ceiling")
    kinds, in0, in1 = packed_gates(xag)
    o = xag.outputs[0]
    cap = n + g + 1
    op = np.zeros(cap, np.int8)
    dst = np.zeros(cap, np.int32)
    s0 = np.zeros(cap, np.int32)
    n0 = np.zeros(cap, np.uint8)
    s1 = np.zeros(cap, np.int32)
    n1 = np.zeros(cap, np.uint8)
    pi = np.zeros(cap, np.int32)
    nreg = np.zeros(1, np.int32)
    rc = N.lib().es_compile(n, g, kinds.ctypes.data, in0.ctypes.data, in1.ctypes.data,
                            o.node * 2 + int(o.neg), op.ctypes.data, dst.ctypes.data,
                            s0.ctypes.data, n0.ctypes.data, s1.ctypes.data, n1.ctypes.data,
                            pi.ctypes.data, nreg.ctypes.data)
    if rc == N.ES_E_TOO_MANY_INPUTS:
        raise TooManyInputs(f"{n} PIs exceeds the {MAX_ES_PIS} ceiling")
    N.check(rc)
    return InstrProgram(op[:rc], dst[:rc], s0[:rc], n0[:rc], s1[:rc], n1[:rc], pi[:rc],
                        int(nreg[0]), n)


class _CancelWatcher:
    """Mirror a Python ``cancel()`` callable into an int32 the engine polls
    between launch slices (the reference polls per batch, es.py:306-309)."""

    def __init__(self, cancel: Callable[[], bool] | None, period_s: float = 0.001):
        self.cancel = cancel
        self.flag = ctypes.c_int32(0)
        self.period = period_s
        self._done = threading.Event()
        self._t = None

    def __enter__(self):
        if self.cancel is not None:
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        return self

    def _poll(self):
        while not self._done.wait(self.period):
            if self.cancel():
                self.flag.value = 1
                return

    def __exit__(self, *exc):
        self._done.set()
        if self._t is not None:
            self._t.join()

    @property
    def address(self):
        return ctypes.addressof(self.flag) if self.cancel is not None else None


def _cofactor_code(cofactor) -> int:
    if isinstance(cofactor, str):
        return N.COFACTOR_MODES[cofactor]
    k = int(cofactor)
    if not 0 <= k <= 5:
        raise ValueError("cofactor must be 'auto', 'none', 'throughput' or 0..5")
    return N.COFACTOR_NONE if k == 0 else k


def _opts(device: int, engine: str, budget: float | None, cancel_addr, slice_ms: float,
          block_threads: int, cofactor="auto", devices: Sequence[int] | None = None,
          jit_parts: int = 0) -> N.EsRunOpts:
    o = N.EsRunOpts()
    o.device = device
    o.engine = N.ENGINES[engine]
    o.budget_s = -1.0 if budget is None else max(float(budget), 0.0)
    o.cancel_flag = cancel_addr
    o.slice_ms = slice_ms
    o.block_threads = block_threads
    o.flags = 0
    o.cofactor_pis = _cofactor_code(cofactor)
    if jit_parts < -1:
        raise ValueError("jit_parts must be >= -1")
    o.jit_parts = jit_parts
    if devices:
        arr = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
        o.n_devices = len(devices)
        o.devices = ctypes.cast(arr, ctypes.c_void_p)
        o._devices_keepalive = arr  # the array must outlive the call
    return o


def _stats_of(r: N.EsResult) -> dict:
    return {"engine": {1: "jit", 2: "interp"}.get(r.engine, "none"),
            "luts": int(r.num_luts), "patterns_swept": int(r.patterns_swept),
            "compile_ms": r.compile_ms, "jit_ms": r.jit_ms, "device_ms": r.device_ms,
            "engine_wall_ms": r.wall_ms, "launches": int(r.launches),
            "regs_per_thread": int(r.regs_per_thread), "cofactor_pis": int(r.cofactor_pis),
            "jit_opt": int(r.jit_opt), "witness_minimal": bool(r.witness_minimal),
            "n_devices": int(r.n_devices), "phases": int(r.phases),
            "phase2_cofactor_pis": int(r.phase2_cofactor_pis) if r.phases == 2 else None,
            "phase2_copies": int(r.phase2_copies) if r.phases == 2 else None,
            "jit_parts": int(r.jit_parts)}


def _to_esresult(r: N.EsResult, num_pis: int) -> EsResult:
    verdict = _VERDICTS[r.verdict]
    if verdict == ES_COUNTEREXAMPLE:
        idx = int(r.witness_index)
        return EsResult(verdict, tuple((idx >> i) & 1 for i in range(num_pis)),
                        int(r.patterns_evaluated), idx, _stats_of(r))
    return EsResult(verdict, None, int(r.patterns_evaluated), None, _stats_of(r))


def run_exhaustive(p, workers: int = 1, budget: float | None = None, cancel=None, *,
                   device: int = 0, engine: str = "auto", slice_ms: float = 20.0,
                   block_threads: int = 0, cofactor="auto",
                   devices: Sequence[int] | None = None, jit_parts: int = 0) -> EsResult:
    """Sweep all 2^num_pis assignments on the GPU (es.py:252-339).

    Returns the minimum-index counterexample (the reference's workers=1
    witness), EXHAUSTED_ZERO, or BUDGET_EXCEEDED when ``budget`` seconds
    elapse or ``cancel()`` turns true first.

    ``cofactor`` (JIT engine): "auto" weighs JIT latency against sweep time
    (and tiers up when a program is re-run), "throughput" picks the fastest
    sweep, "none" or 0 disables, 1..5 forces that many cofactor PIs.  The
    result is the same for every setting.

    ``devices``: sweep on these CUDA ordinals at once (the reference's
    ``workers``, es.py:272-331, as GPUs): chunks of the pattern space are
    dealt round-robin, one host thread drives each device, and one minimum
    word shared over NVLink stops every GPU once a smaller pattern cannot
    exist.  ``"all"`` = every visible GPU.  Default: ``device`` alone.

    ``jit_parts`` (JIT engine): 0 lets the policy pick the build -- for a
    cold program the direct-SASS kernel (es_sass.cpp: the body encoded by the
    library itself, no ptxas) or a body split into phases that ptxas compiles
    on parallel host threads (es_split.cpp), tiering up to ptxas -O3 as the
    program is re-run; 1 keeps one straight-line ptxas body, >= 2 forces that
    many phases, -1 forces direct SASS.
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    prog = as_program(p)
    # a constant output is decided before the budget is looked at (es.py:265-270);
    # otherwise a spent budget or a raised cancel stops before the first batch
    if prog.src0[-1] >= 0:
        if budget is not None and budget <= 0:
            return EsResult(BUDGET_EXCEEDED, patterns_evaluated=0)
        if cancel is not None and cancel():
            return EsResult(BUDGET_EXCEEDED, patterns_evaluated=0)
    res = N.EsResult()
    with _CancelWatcher(cancel) as cw:
        opts = _opts(device, engine, budget, cw.address, slice_ms, block_threads, cofactor,
                     _devices(devices), jit_parts)
        N.check(N.lib().es_run(ctypes.byref(prog.as_struct()), ctypes.byref(opts),
                               ctypes.byref(res)))
    return _to_esresult(res, prog.num_pis)


def _recheck(xag, witness) -> int:
    """The witness re-check (es.py:360-361) natively (es_xag_eval); XAGs over
    64 PIs (never ES-eligible) fall back to the direct evaluation."""
    if xag.num_pis > 64 or len(xag.outputs) != 1:
        return evaluate(xag, witness)
    kind, in0, in1 = packed_gates(xag)
    o = xag.outputs[0]
    idx = sum(int(b) << i for i, b in enumerate(witness))
    return N.check(N.lib().es_xag_eval(xag.num_pis, len(xag.gates), kind.ctypes.data, in0.ctypes.data,
                                       in1.ctypes.data, o.node * 2 + int(o.neg), idx))


def device_count() -> int:
    """Visible CUDA devices (0 without a driver)."""
    n = ctypes.c_int32()
    N.check(N.lib().es_device_count(ctypes.byref(n)))
    return n.value


def _devices(devices) -> list[int] | None:
    if devices is None:
        return None
    if isinstance(devices, str):
        if devices != "all":
            raise ValueError("devices must be a sequence of ordinals or 'all'")
        n = device_count()
        if n < 1:
            raise N.NativeError(N.ES_E_NO_DEVICE, "no CUDA device visible")
        return list(range(n))
    d = [int(x) for x in devices]
    if not d:
        raise ValueError("devices must not be empty")
    return d


def es_check(sm, workers: int = 1, budget: float | None = None, cancel=None, *,
             device: int = 0, engine: str = "auto", cofactor="auto",
             devices: Sequence[int] | str | None = None, jit_parts: int = 0) -> CheckResult:
    """Compile and sweep a sub-miter (es.py:342-365); witnesses are re-checked
    by direct evaluation and a mismatch raises AssertionError."""
    t0 = time.monotonic()
    try:
        prog = compile_program(sm.circuit)
    except TooManyInputs:
        return CheckResult(UNKNOWN, reason="ineligible", engine="es")
    r = run_exhaustive(prog, workers=workers, budget=budget, cancel=cancel, device=device,
                       engine=engine, cofactor=cofactor, devices=devices, jit_parts=jit_parts)
    stats = {"patterns": r.patterns_evaluated, "registers": prog.num_registers,
             "wall_time": time.monotonic() - t0, **r.stats}
    if r.verdict == EXHAUSTED_ZERO:
        return CheckResult(EQUIVALENT, engine="es", stats=stats)
    if r.verdict == ES_COUNTEREXAMPLE:
        if _recheck(sm.circuit, r.witness) != 1:
            raise AssertionError("exhaustive-simulation witness failed re-check")
        return CheckResult(COUNTEREXAMPLE, witness=r.witness, engine="es", stats=stats)
    reason = "cancelled" if (cancel is not None and cancel()) else "timeout"
    return CheckResult(UNKNOWN, reason=reason, engine="es", stats=stats)


def run_exhaustive_batch(progs: Sequence, budget: float | None = None, cancel=None, *,
                         device: int = 0) -> list[EsResult]:
    """One interpreter launch over many programs (sweep's sub-miter stream)."""
    ps = [as_program(p) for p in progs]
    if not ps:
        return []
    # budget <= 0 is decided natively, after each job's constant-rail check (es.py:265-270)
    arr = (N.EsProg * len(ps))(*[p.as_struct() for p in ps])
    outs = (N.EsResult * len(ps))()
    with _CancelWatcher(cancel) as cw:
        # "auto": programs too wide for the interpreter's shared memory run on K1
        opts = _opts(device, "auto", budget, cw.address, 20.0, 0)
        N.check(N.lib().es_run_batch(len(ps), arr, ctypes.byref(opts), outs))
    return [_to_esresult(outs[i], ps[i].num_pis) for i in range(len(ps))]


def es_check_batch(sms: Iterable, budget: float | None = None, cancel=None, *,
                   device: int = 0) -> list[CheckResult]:
    """Batched ``es_check`` over many sub-miters (config 4)."""
    sms = list(sms)
    t0 = time.monotonic()
    results: list[CheckResult | None] = [None] * len(sms)
    progs, where = [], []
    for i, sm in enumerate(sms):
        try:
            progs.append(compile_program(sm.circuit))
            where.append(i)
        except TooManyInputs:
            results[i] = CheckResult(UNKNOWN, reason="ineligible", engine="es")
    rs = run_exhaustive_batch(progs, budget=budget, cancel=cancel, device=device)
    wall = time.monotonic() - t0
    for i, p, r in zip(where, progs, rs):
        stats = {"patterns": r.patterns_evaluated, "registers": p.num_registers,
                 "wall_time": wall, **r.stats}
        if r.verdict == EXHAUSTED_ZERO:
            results[i] = CheckResult(EQUIVALENT, engine="es", stats=stats)
        elif r.verdict == ES_COUNTEREXAMPLE:
            if _recheck(sms[i].circuit, r.witness) != 1:
                raise AssertionError("exhaustive-simulation witness failed re-check")
            results[i] = CheckResult(COUNTEREXAMPLE, witness=r.witness, engine="es", stats=stats)
        else:
            reason = "cancelled" if (cancel is not None and cancel()) else "timeout"
            results[i] = CheckResult(UNKNOWN, reason=reason, engine="es", stats=stats)
    return results  # type: ignore[return-value]


# --- engine introspection (tests, profiling) --------------------------------

def map_stats(p, k: int = 0) -> dict:
    """K1 mapping of ``p`` with ``k`` cofactor PIs: LUTs per iteration (2^k
    words), schedule peak live set, cone gates, the cofactor PIs."""
    prog = as_program(p)
    luts, live, gates = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    pis = (ctypes.c_int32 * 8)()
    N.check(N.lib().es_map_stats_k(ctypes.byref(prog.as_struct()), k, ctypes.byref(luts),
                                   ctypes.byref(live), ctypes.byref(gates), pis))
    return {"luts": luts.value, "peak_live": live.value, "gates": gates.value,
            "cofactor_pis": list(pis[:k])}


def map_stats_restricted(p, k: int, copies: int) -> dict:
    """The k-PI cofactor variant restricted to copies 0..copies-1 (the second
    phase of a non-equivalent search): LUTs per iteration, peak live set."""
    prog = as_program(p)
    luts, live = ctypes.c_int32(), ctypes.c_int32()
    N.check(N.lib().es_map_stats_kc(ctypes.byref(prog.as_struct()), k, copies, ctypes.byref(luts),
                                    ctypes.byref(live)))
    return {"luts": luts.value, "peak_live": live.value}


def map_eval_restricted(p, w0: int, nw: int, k: int, copies: int) -> np.ndarray:
    """CPU model of the restricted variant (0 for words of other copies)."""
    prog = as_program(p)
    out = np.zeros(nw, dtype=np.uint32)
    N.check(N.lib().es_map_eval_kc(ctypes.byref(prog.as_struct()), k, copies, w0, nw,
                                   out.ctypes.data))
    return out


def map_pipes(p, k: int = 0) -> dict:
    """K1 body ops per iteration: LOP3 (ALU pipe) and IMAD (FMA pipe)."""
    prog = as_program(p)
    l, i = ctypes.c_int32(), ctypes.c_int32()
    N.check(N.lib().es_map_pipes_k(ctypes.byref(prog.as_struct()), k, ctypes.byref(l),
                                   ctypes.byref(i)))
    return {"lop3": l.value, "imad": i.value}


def map_eval(p, w0: int, nw: int, k: int = 0) -> np.ndarray:
    """CPU model of the mapped kernel body: output words [w0, w0+nw) (full
    word indices; with k cofactor PIs each word comes from its copy)."""
    prog = as_program(p)
    out = np.zeros(nw, dtype=np.uint32)
    N.check(N.lib().es_map_eval_k(ctypes.byref(prog.as_struct()), k, w0, nw, out.ctypes.data))
    return out


def k2_stats(p) -> dict:
    """The K2 interpreter's program for ``p``: gates, slots, stores, forwards."""
    prog = as_program(p)
    v = [ctypes.c_int32() for _ in range(4)]
    N.check(N.lib().es_k2_stats(ctypes.byref(prog.as_struct()), *[ctypes.byref(x) for x in v]))
    return {"gates": v[0].value, "slots": v[1].value, "stores": v[2].value,
            "acc_reads": v[3].value}


def k2_eval(p, w0: int, nw: int, k: int | None = None) -> np.ndarray:
    """CPU model of the K2 interpreter: output words [w0, w0+nw) (full word
    indices).  ``k``: forced cofactor PIs; None = the depth K2 picks."""
    prog = as_program(p)
    out = np.zeros(nw, dtype=np.uint32)
    if k is None:
        N.check(N.lib().es_k2_eval(ctypes.byref(prog.as_struct()), w0, nw, out.ctypes.data))
    else:
        N.check(N.lib().es_k2_eval_k(ctypes.byref(prog.as_struct()), k, w0, nw, out.ctypes.data))
    return out


def k2_cofactor_pis(p) -> int:
    """Cofactor depth the K2 interpreter picks for ``p``."""
    return N.check(N.lib().es_k2_cofactor_pis(ctypes.byref(as_program(p).as_struct())))


def emit_ptx(p, block_threads: int = 256, k: int = 0) -> str:
    prog = as_program(p)
    L = N.lib()
    n = N.check(L.es_emit_ptx_k(ctypes.byref(prog.as_struct()), k, block_threads, None, 0))
    buf = ctypes.create_string_buffer(n)
    N.check(L.es_emit_ptx_k(ctypes.byref(prog.as_struct()), k, block_threads, buf, n))
    return buf.value.decode()


def jit_check(p, block_threads: int = 256, k: int = 0) -> dict:
    """PTX -> SASS for ``p`` without a GPU: cubin size, registers, spills."""
    prog = as_program(p)
    regs, spill = ctypes.c_int32(), ctypes.c_int32()
    log = ctypes.create_string_buffer(1 << 16)
    n = N.check(N.lib().es_jit_check_k(ctypes.byref(prog.as_struct()), k, block_threads,
                                       ctypes.byref(regs), ctypes.byref(spill), log, 1 << 16))
    return {"cubin_bytes": n, "regs": regs.value, "spill_bytes": spill.value,
            "log": log.value.decode(errors="replace")}
