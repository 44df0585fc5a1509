"""Shared-memory overflow slots of the K1 body (csrc/es_spill.cpp; north_star
(2)): the rewritten body computes exactly what the register-only body does.

A small interpreter runs the emitted PTX body (the LOP3/IMAD block K1
splices into its skeleton) over numpy vectors -- one element per thread,
shared memory as a flat array addressed like the kernel's slot file -- for
the plain body and for the spilled one at several register budgets, and
both are compared with the CPU model of the mapped program (es.map_eval).
No GPU needed; the GPU parity of the spilled kernel is in
tests/test_spill_gpu.py."""
import ctypes
import re

import numpy as np
import pytest

from paper_2512_06627_b200 import _native as N
from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M

M32 = np.uint64(0xFFFFFFFF)


def body_of(p, k, budget, threads):
    L = N.lib()
    slots = ctypes.c_int32()
    n = N.check(L.es_emit_body_k(ctypes.byref(p.as_struct()), k, budget, threads, ctypes.byref(slots), None, 0))
    buf = ctypes.create_string_buffer(n)
    N.check(L.es_emit_body_k(ctypes.byref(p.as_struct()), k, budget, threads, ctypes.byref(slots), buf, n))
    return buf.value.decode(), slots.value


def run_body(text, wlo, whi, threads, slots):
    """Interpret the body for `threads` threads (numpy uint32 vectors)."""
    T = len(wlo)
    R = {"%lo": wlo.astype(np.uint32), "%hi": whi.astype(np.uint32), "%one": np.ones(T, np.uint32),
         "%tid.x": np.arange(T, dtype=np.uint32) % threads, "es_slots": np.zeros(T, np.uint32)}
    smem = np.zeros((max(slots, 1) * threads + threads) * 1, np.uint32)
    pred = {}

    def val(x):
        if x.startswith("%") or x == "es_slots":
            return R[x]
        return np.full(T, int(x) & 0xFFFFFFFF, np.uint32)

    def sval(x):
        return val(x).astype(np.int32).astype(np.int64)

    for line in text.splitlines():
        line = line.strip()
        if not line or line[0] in ".{}/":
            continue
        op, rest = line.split(None, 1)
        ops = [t.strip() for t in rest.rstrip(";").split(",")]
        d = ops[0]
        if op == "lop3.b32":
            a, b, c = (val(x).astype(np.uint64) for x in ops[1:4])
            tt = int(ops[4])
            r = np.zeros(T, np.uint64)
            for i in range(8):
                if (tt >> i) & 1:
                    r |= ((a if i & 4 else ~a) & (b if i & 2 else ~b) & (c if i & 1 else ~c)) & M32
            R[d] = r.astype(np.uint32)
        elif op == "mad.lo.s32":
            R[d] = ((sval(ops[1]) * sval(ops[2]) + sval(ops[3])) & 0xFFFFFFFF).astype(np.uint32)
        elif op in ("mul.lo.s32", "mul.lo.u32"):
            R[d] = ((val(ops[1]).astype(np.uint64) * val(ops[2]).astype(np.uint64)) & M32).astype(np.uint32)
        elif op == "mul.hi.s32":
            R[d] = ((sval(ops[1]) * sval(ops[2])) >> 32).astype(np.int64).astype(np.uint32)
        elif op in ("mov.b32", "mov.u32"):
            R[d] = val(ops[1]).copy()
        elif op == "neg.s32":
            R[d] = (-sval(ops[1]) & 0xFFFFFFFF).astype(np.uint32)
        elif op == "not.b32":
            R[d] = ~val(ops[1])
        elif op == "shl.b32":
            R[d] = (val(ops[1]).astype(np.uint64) << np.uint64(int(ops[2])) & M32).astype(np.uint32)
        elif op == "shr.s32":
            R[d] = (sval(ops[1]) >> int(ops[2])).astype(np.uint32)
        elif op in ("add.u32", "add.s32"):
            R[d] = ((val(ops[1]).astype(np.uint64) + val(ops[2]).astype(np.uint64)) & M32).astype(np.uint32)
        elif op == "setp.eq.b32":
            pred[d] = val(ops[1]) == val(ops[2])
        elif op == "selp.b32":
            R[d] = np.where(pred[ops[3]], val(ops[1]), val(ops[2])).astype(np.uint32)
        elif op == "ld.shared.b32":
            m = re.fullmatch(r"\[(%\w+)\+(\d+)\]", ops[1])
            R[d] = smem[(R[m.group(1)] + int(m.group(2))) // 4]
        elif op == "st.shared.b32":
            m = re.fullmatch(r"\[(%\w+)\+(\d+)\]", ops[0])
            smem[(R[m.group(1)] + int(m.group(2))) // 4] = val(ops[1])
        else:
            raise AssertionError(f"interpreter: unknown op {op}")
    return R


def check(x, k, budget, threads=128, nwords=256, seed=0):
    p = es.compile_program(x)
    plain, s0 = body_of(p, k, 0, threads)
    spilled, s1 = body_of(p, k, budget, threads)
    assert s0 == 0
    n_kernel_bits = max(p.num_pis - 5 - k, 0)
    rng = np.random.default_rng(seed)
    # kernel word indices (cofactor PIs excluded); one warp-sized group per CTA
    w = rng.integers(0, 1 << n_kernel_bits, size=threads, dtype=np.uint64) if n_kernel_bits else \
        np.zeros(threads, np.uint64)
    lo, hi = (w & M32).astype(np.uint32), (w >> np.uint64(32)).astype(np.uint32)
    a = run_body(plain, lo, hi, threads, 0)
    b = run_body(spilled, lo, hi, threads, s1)
    outs = ("%o", "%c") if "%c" in plain else ("%o",)
    for o in outs:
        np.testing.assert_array_equal(a[o], b[o])
    return p, a, s1, spilled


@pytest.mark.parametrize("k,budget", [(0, 24), (0, 60), (2, 30), (3, 40), (4, 64)])
def test_spilled_body_equals_register_body(k, budget):
    x = M.gen_multiplier_miter(8, "array", "booth")
    _, _, slots, text = check(x, k, budget)
    assert slots > 0 and "st.shared.b32" in text and "ld.shared.b32" in text


def test_spilled_body_matches_cpu_model_on_fault():
    """The register-only body on a failing miter equals es.map_eval (the CPU
    model of the mapped program), and so does the spilled body."""
    x = M.flip_gate(M.gen_multiplier_miter(8, "array", "booth"), 120)
    p = es.compile_program(x)
    k, threads = 0, 128
    plain, _ = body_of(p, k, 0, threads)
    spilled, slots = body_of(p, k, 20, threads)
    w = np.arange(threads, dtype=np.uint64) * np.uint64(7) % np.uint64(1 << (p.num_pis - 5))
    lo, hi = (w & M32).astype(np.uint32), (w >> np.uint64(32)).astype(np.uint32)
    ref = np.array([es.map_eval(p, int(v), 1, k)[0] for v in w], np.uint32)
    valid = np.uint32(0xFFFFFFFF)
    for text, s in ((plain, 0), (spilled, slots)):
        got = run_body(text, lo, hi, threads, s)["%o"] & valid
        np.testing.assert_array_equal(got, ref)
    assert ref.any()  # the fault is visible on these words


def test_budget_bounds_register_live_set_and_slots_fit():
    """mult16 at 4 cofactor PIs: the rewrite keeps the live set within the
    budget and needs fewer slots than values it moves out."""
    p = es.compile_program(M.gen_multiplier_miter(16, "array", "booth"))
    _, slots_240 = body_of(p, 4, 240, 256)
    _, slots_140 = body_of(p, 4, 140, 128)
    assert 0 < slots_240 < slots_140
    # 12 warps per SM: three 128-thread CTAs of slots*128*4 bytes fit 228 KB
    assert 3 * slots_140 * 128 * 4 <= 228 * 1024
