"""K1 JIT on the CPU: spliced PTX compiles to sm_100a SASS in process, with
no spills, for every configuration miter (no GPU needed)."""
import pytest

from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M


@pytest.mark.parametrize("name,x", [
    ("adder8", M.gen_adder_miter(8)),
    ("mult12", M.gen_multiplier_miter(12, "array", "wallace")),
    ("mult16", M.gen_multiplier_miter(16, "array", "booth")),
    ("mult16_fault", M.flip_gate(M.gen_multiplier_miter(16, "array", "booth"), 1953)),
])
def test_jit_compiles_without_spills(name, x):
    j = es.jit_check(es.compile_program(x), block_threads=128)
    assert j["cubin_bytes"] > 0
    assert 0 < j["regs"] <= 255
    assert j["spill_bytes"] == 0, j["log"]


def test_ptx_has_one_body_and_lop3():
    p = es.compile_program(M.gen_multiplier_miter(6, "array", "booth"))
    ptx = es.emit_ptx(p, 256)
    assert ".entry es_k1" in ptx and ".target sm_100a" in ptx
    # every LUT is one LOP3 (ALU pipe) or one IMAD (FMA pipe, f(x, word PI))
    luts = es.map_stats(p)["luts"]
    n_mad = sum(1 for ln in ptx.splitlines() if ln.startswith("mad.lo.s32 %esq"))
    assert ptx.count("lop3.b32") + n_mad == luts and n_mad > 0
    assert "ES_BODY" not in ptx
    assert "atom.sys.global.min.u64" in ptx or "atom.global.sys.min.u64" in ptx


def test_unsupported_block_size():
    p = es.compile_program(M.gen_multiplier_miter(3, "array", "diagonal"))
    with pytest.raises(Exception):
        es.emit_ptx(p, 96)


def test_throughput_kernel_mult16_k4_has_no_spills():
    """The bench's kernel (mult16, 4 cofactor PIs, 256-thread CTAs): with the
    copies visited in bit-reversed order the schedule's live set is ~212
    values and ptxas fits it in 255 registers without spilling (the index
    order needed 358 values and spilled ~1 KB per thread)."""
    from paper_2512_06627_b200 import miter as M

    p = es.compile_program(M.gen_multiplier_miter(16, "array", "booth"))
    assert es.map_stats(p, 4)["peak_live"] <= 230
    j = es.jit_check(p, block_threads=256, k=4)
    assert j["spill_bytes"] == 0, j["log"]


@pytest.mark.parametrize("k,parts", [(0, 2), (0, 6), (2, 4)])
def test_split_build_compiles_and_links(k, parts):
    """The split build (es_split.cpp): phase modules compile relocatable and
    nvJitLink joins them with the skeleton, with no GPU."""
    import ctypes

    from paper_2512_06627_b200 import _native as N

    p = es.compile_program(M.gen_multiplier_miter(12, "array", "wallace"))
    regs, smem, slots, loads = (ctypes.c_int32() for _ in range(4))
    ms = ctypes.c_double()
    n = N.check(N.lib().es_jit_check_split(ctypes.byref(p.as_struct()), k, parts, 128, ctypes.byref(regs),
                                           ctypes.byref(smem), ctypes.byref(slots), ctypes.byref(loads),
                                           ctypes.byref(ms)))
    assert n > 0
    assert slots.value > 0 and smem.value == slots.value * 128 * 4 and loads.value >= slots.value - 2
