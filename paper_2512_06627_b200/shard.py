"""Multi-GPU exact simulation: one process per GPU, the 2^n input space
sharded across ranks.

Chunks of the pattern space are dealt round-robin to ranks (chunk % world ==
rank) and swept in increasing order by each rank's K1 kernel.  The only
exchange is the 8-byte minimum failing pattern: after every launch slice the
ranks all-reduce it with MIN over NCCL, so a counterexample found by any GPU
stops every GPU at the next chunk claim (global early termination), and the
final value is the minimum-index witness -- bit-exact with the reference's
single-worker sweep (es.py:297-320) for any world size.

torch is used only as plumbing: device memory for the 8-byte word, the
stream, and torch.distributed's NCCL all-reduce.
"""

from __future__ import annotations

import ctypes

from . import _native as N
from .es import (BUDGET_EXCEEDED, ES_COUNTEREXAMPLE, EXHAUSTED_ZERO, EsResult, as_program,
                 _opts)


class Session:
    """A program JIT-compiled for one device, launchable on any stream."""

    def __init__(self, prog, device: int = 0, block_threads: int = 0, cofactor="throughput"):
        self.prog = as_program(prog)
        self.device = device
        # sessions serve repeated / long sharded sweeps: default to the fastest
        # K1 variant (es_run_opts.cofactor_pis); the JIT is paid once per session
        opts = _opts(device, "jit", None, None, 20.0, block_threads, cofactor)
        h = ctypes.c_void_p()
        N.check(N.lib().es_session_open(ctypes.byref(self.prog.as_struct()), ctypes.byref(opts),
                                        ctypes.byref(h)))
        self._h = h
        nc, ppc = ctypes.c_uint64(), ctypes.c_uint64()
        luts, regs = ctypes.c_int32(), ctypes.c_int32()
        N.check(N.lib().es_session_geometry(h, ctypes.byref(nc), ctypes.byref(ppc),
                                            ctypes.byref(luts), ctypes.byref(regs)))
        self.n_chunks = nc.value
        self.patterns_per_chunk = ppc.value
        self.num_luts = luts.value
        self.regs_per_thread = regs.value

    def launch(self, stream: int, best_ptr: int, chunk_begin: int, chunk_end: int,
               rank: int = 0, world: int = 1) -> None:
        N.check(N.lib().es_session_launch(self._h, ctypes.c_void_p(stream), ctypes.c_void_p(best_ptr),
                                          chunk_begin, chunk_end, rank, world))

    def close(self) -> None:
        if self._h:
            N.lib().es_session_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rank_chunks(chunk_begin: int, chunk_end: int, rank: int, world: int) -> range:
    """Chunks one rank sweeps in a launch over [chunk_begin, chunk_end):
    its residue class mod world.  Mirrors session_launch (es_runtime.cu)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard")
    first = chunk_begin + (rank - chunk_begin % world) % world
    return range(first, chunk_end, world)


def slice_bounds(n_chunks: int, slices: int) -> list[int]:
    """Launch-slice boundaries; a MIN all-reduce follows every slice."""
    s = max(1, min(slices, n_chunks))
    return [n_chunks * i // s for i in range(s + 1)]


def sharded_loop(n_chunks: int, slices: int, launch, reduce) -> int:
    """The rank-side schedule of a sharded sweep: launch a slice, reduce the
    minimum across ranks, repeat.  Returns the number of slices."""
    b = slice_bounds(n_chunks, slices)
    for i in range(len(b) - 1):
        launch(b[i], b[i + 1])
        reduce()
    return len(b) - 1


_sessions: dict[tuple[int, int], Session] = {}


def session_for(prog, device: int, cofactor="throughput") -> Session:
    p = as_program(prog)
    key = (hash(bytes(p.op) + bytes(p.dst) + bytes(p.src0) + bytes(p.src1) + bytes(p.neg0)
                + bytes(p.neg1) + bytes(p.pi)) ^ p.num_pis, device, str(cofactor))
    s = _sessions.get(key)
    if s is None:
        s = _sessions[key] = Session(p, device, cofactor=cofactor)
    return s


def sweep_sharded(prog, group=None, device: int | None = None, slices: int | None = None,
                  best=None, cofactor="throughput") -> EsResult:
    """run_exhaustive sharded over the ranks of ``group`` (collective call).

    Every rank must call it with the same program.  ``slices`` launch slices
    separate the MIN all-reduces (early-termination granularity); default 1
    on a single rank, 8 otherwise.  Returns the same EsResult on every rank.
    """
    import torch
    import torch.distributed as dist

    p = as_program(prog)
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    dev = torch.cuda.current_device() if device is None else device
    last = len(p) - 1
    if p.src0[last] < 0:  # constant rail, es.py:265-270
        if p.neg0[last]:
            return EsResult(ES_COUNTEREXAMPLE, (0,) * p.num_pis, 0, 0)
        return EsResult(EXHAUSTED_ZERO, None, 1 << p.num_pis)
    sess = session_for(p, dev, cofactor)
    sentinel = 1 << p.num_pis
    if best is None:
        best = torch.empty(1, dtype=torch.int64, device=f"cuda:{dev}")
    best.fill_(sentinel)
    stream = torch.cuda.current_stream(dev).cuda_stream
    S = slices or (1 if world == 1 else 8)

    def launch(lo: int, hi: int) -> None:
        sess.launch(stream, best.data_ptr(), lo, hi, rank, world)

    def reduce() -> None:
        if world > 1:
            dist.all_reduce(best, op=dist.ReduceOp.MIN, group=group)

    sharded_loop(sess.n_chunks, S, launch, reduce)
    b = int(best.item())
    if b < sentinel:
        lo = min(p.num_pis, 14)
        return EsResult(ES_COUNTEREXAMPLE, tuple((b >> i) & 1 for i in range(p.num_pis)),
                        ((b >> lo) + 1) << lo, b)
    return EsResult(EXHAUSTED_ZERO, None, sentinel)


def alu_peak(device: int = 0) -> tuple[float, float]:
    """Measured lane-LOP3/s of the device (and the microbenchmark's ms)."""
    v, ms = ctypes.c_double(), ctypes.c_double()
    N.check(N.lib().es_alu_peak(device, ctypes.byref(v), ctypes.byref(ms)))
    return v.value, ms.value


def fma_peak(device: int = 0) -> tuple[float, float]:
    """Measured lane-IMAD/s of the device's FMA pipe (and the ms)."""
    v, ms = ctypes.c_double(), ctypes.c_double()
    N.check(N.lib().es_fma_peak(device, ctypes.byref(v), ctypes.byref(ms)))
    return v.value, ms.value


def smem_peak(device: int = 0) -> tuple[float, float]:
    """Measured shared-memory load bytes/s of the device (and the ms)."""
    v, ms = ctypes.c_double(), ctypes.c_double()
    N.check(N.lib().es_smem_peak(device, ctypes.byref(v), ctypes.byref(ms)))
    return v.value, ms.value


def es_check_sharded(sm, group=None, device: int | None = None,
                     slices: int | None = None, cofactor="throughput"):
    """``es_check`` (es.py:342-365) with the sweep sharded over ``group``."""
    import time

    from .es import TooManyInputs, compile_program
    from .miter import evaluate
    from .verdict import COUNTEREXAMPLE, EQUIVALENT, UNKNOWN, CheckResult

    t0 = time.monotonic()
    try:
        prog = compile_program(sm.circuit)
    except TooManyInputs:
        return CheckResult(UNKNOWN, reason="ineligible", engine="es")
    r = sweep_sharded(prog, group, device, slices, cofactor=cofactor)
    stats = {"patterns": r.patterns_evaluated, "registers": prog.num_registers,
             "wall_time": time.monotonic() - t0}
    if r.verdict == EXHAUSTED_ZERO:
        return CheckResult(EQUIVALENT, engine="es", stats=stats)
    if evaluate(sm.circuit, r.witness) != 1:
        raise AssertionError("exhaustive-simulation witness failed re-check")
    return CheckResult(COUNTEREXAMPLE, witness=r.witness, engine="es", stats=stats)


class PeerBest:
    """The NVLink-native exchange: minimum words in rank 0's
    device memory, mapped into every rank through CUDA IPC.  Every rank's
    kernel atomicMin's (system scope) into the verdict's word and reads it at
    each chunk claim, so a counterexample found on any GPU stops every GPU at
    its next chunk -- no collective on the data path.  Each word carries an
    arrival counter: after its sweep a rank's stream runs es_peer_arrive_wait
    (a one-thread kernel: count in, wait on the device for all ranks, copy
    the final minimum out), so a verdict needs no host barrier and the host
    can queue verdicts back to back.  Three words rotate: rank 0 re-arms the
    word of verdict s+1 on its stream while verdict s runs; that word was
    last used by verdict s-2, whose device barrier every rank passed before
    any rank could finish verdict s-1.  Words are armed with all-ones (no
    pattern index reaches it), so one PeerBest serves programs of any PI
    count.  Collective constructor (every rank of ``group``)."""

    NONE = 0xFFFFFFFFFFFFFFFF  # "no counterexample yet"
    WORDS = 3

    def __init__(self, group=None, device: int | None = None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.device = torch.cuda.current_device() if device is None else device
        self.ptrs = []
        self._step = 0
        L = N.lib()
        for _ in range(self.WORDS):
            ptr = ctypes.c_void_p()
            handle = (ctypes.c_uint8 * 64)()
            if self.rank == 0:
                # zero-filled: arrival counter 0; the word is armed before it is shared
                N.check(L.es_ipc_alloc(self.device, ctypes.byref(ptr), handle))
                N.check(L.es_word_write(self.device, ptr, self.NONE))
            box = [bytes(handle)]
            if self.world > 1:
                dist.broadcast_object_list(box, src=0, group=group)
            if self.rank != 0:
                h = (ctypes.c_uint8 * 64).from_buffer_copy(box[0])
                N.check(L.es_ipc_open(self.device, h, ctypes.byref(ptr)))
            self.ptrs.append(ptr)
        if self.world > 1:
            dist.barrier(group=group)  # every rank has mapped the words

    def write(self, k: int, value: int) -> None:
        N.check(N.lib().es_word_write(self.device, self.ptrs[k], value))

    def read(self, k: int) -> int:
        v = ctypes.c_uint64()
        N.check(N.lib().es_word_read(self.device, self.ptrs[k], ctypes.byref(v)))
        return v.value

    def close(self) -> None:
        """Collective: no rank may still be using rank 0's words."""
        import torch
        import torch.distributed as dist

        torch.cuda.synchronize(self.device)
        if self.world > 1:
            dist.barrier(group=self.group)
        for p in self.ptrs:
            if p:
                N.lib().es_ipc_close(self.device, p, 1 if self.rank == 0 else 0)
        self.ptrs = []


def _constant_rail(p) -> EsResult | None:
    last = len(p) - 1
    if p.src0[last] < 0:  # constant rail, es.py:265-270
        if p.neg0[last]:
            return EsResult(ES_COUNTEREXAMPLE, (0,) * p.num_pis, 0, 0)
        return EsResult(EXHAUSTED_ZERO, None, 1 << p.num_pis)
    return None


def sweep_peer_async(prog, peer: PeerBest, out_ptr: int, device: int | None = None,
                     cofactor="throughput", stream: int | None = None) -> None:
    """Queue one sharded verdict on ``stream`` (default: torch's current
    stream) without host synchronisation: this rank's sweep over its residue
    class of chunks, then the device-side barrier that writes the final
    minimum (all-ones: none) to the 8-byte device buffer at ``out_ptr``.
    Collective: every rank queues the same programs in the same order."""
    import torch

    p = as_program(prog)
    dev = peer.device if device is None else device
    sess = session_for(p, dev, cofactor)
    st = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
    k = peer._step % peer.WORDS
    peer._step += 1
    L = N.lib()
    if peer.rank == 0:  # the next verdict's word: last used two verdicts ago
        N.check(L.es_peer_arm(ctypes.c_void_p(st), peer.ptrs[(k + 1) % peer.WORDS]))
    sess.launch(st, peer.ptrs[k].value, 0, sess.n_chunks, peer.rank, peer.world)
    N.check(L.es_peer_arrive_wait(ctypes.c_void_p(st), peer.ptrs[k], peer.world,
                                  ctypes.c_void_p(out_ptr)))


def peer_result(p, b: int) -> EsResult:
    """EsResult of a verdict whose final minimum word is ``b``."""
    p = as_program(p)
    sentinel = 1 << p.num_pis
    if b < sentinel:
        lo = min(p.num_pis, 14)
        return EsResult(ES_COUNTEREXAMPLE, tuple((b >> i) & 1 for i in range(p.num_pis)),
                        ((b >> lo) + 1) << lo, b)
    return EsResult(EXHAUSTED_ZERO, None, sentinel)


def sweep_peer(prog, peer: PeerBest, group=None, device: int | None = None,
               cofactor="throughput") -> EsResult:
    """run_exhaustive sharded over ``group`` with the shared peer word
    (collective call; same program on every rank).  One launch per rank over
    its residue class of chunks, the device-side barrier, one 8-byte read."""
    import torch

    p = as_program(prog)
    rail = _constant_rail(p)
    if rail is not None:
        return rail
    dev = peer.device if device is None else device
    out = torch.empty(1, dtype=torch.int64, device=f"cuda:{dev}")
    sweep_peer_async(p, peer, out.data_ptr(), dev, cofactor)
    return peer_result(p, int(out.item()) & 0xFFFFFFFFFFFFFFFF)


def es_check_peer(sm, peer: PeerBest, group=None, device: int | None = None,
                  cofactor="throughput"):
    """``es_check`` (es.py:342-365) sharded with the shared peer word."""
    import time

    from .es import TooManyInputs, compile_program
    from .miter import evaluate
    from .verdict import COUNTEREXAMPLE, EQUIVALENT, UNKNOWN, CheckResult

    t0 = time.monotonic()
    try:
        prog = compile_program(sm.circuit)
    except TooManyInputs:
        return CheckResult(UNKNOWN, reason="ineligible", engine="es")
    r = sweep_peer(prog, peer, group, device, cofactor=cofactor)
    stats = {"patterns": r.patterns_evaluated, "registers": prog.num_registers,
             "wall_time": time.monotonic() - t0}
    if r.verdict == EXHAUSTED_ZERO:
        return CheckResult(EQUIVALENT, engine="es", stats=stats)
    if evaluate(sm.circuit, r.witness) != 1:
        raise AssertionError("exhaustive-simulation witness failed re-check")
    return CheckResult(COUNTEREXAMPLE, witness=r.witness, engine="es", stats=stats)
