"""The C-ABI library loads without a GPU and exports every symbol its header
declares; host-only entry points work; compute entry points fail loudly
(never fall back) when no device is visible."""
import ctypes
import os
import re

import pytest

from paper_2512_06627_b200 import _native as N
from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "es_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(es_[a-z_0-9]+)\s*\(", text))


def test_header_and_exports_agree():
    assert header_functions() == set(N.EXPORTS)


def test_library_exports_every_symbol():
    L = ctypes.CDLL(N.LIB_PATH)
    for name in header_functions():
        assert hasattr(L, name), name


def test_version_and_errors():
    assert b"sm_100a" in N.lib().es_version()
    b = ctypes.c_int32()
    rc = N.lib().es_map_stats(None, ctypes.byref(b), None, None)
    assert rc == N.ES_E_BAD_PROGRAM and N.last_error()


def test_bad_programs_rejected():
    p = es.compile_program(M.gen_multiplier_miter(3, "array", "diagonal"))
    bad = es.InstrProgram(p.op[:-1], p.dst[:-1], p.src0[:-1], p.neg0[:-1], p.src1[:-1],
                          p.neg1[:-1], p.pi[:-1], p.num_registers, p.num_pis)
    with pytest.raises(N.NativeError):
        es.map_stats(bad)                     # no OUTPUT
    src = p.src0.copy()
    src[len(p) // 2] = p.num_registers + 3    # undefined register
    bad = es.InstrProgram(p.op, p.dst, src, p.neg0, p.src1, p.neg1, p.pi, p.num_registers,
                          p.num_pis)
    with pytest.raises(N.NativeError):
        es.map_stats(bad)


def test_workers_validated():
    p = es.compile_program(M.gen_multiplier_miter(3, "array", "diagonal"))
    with pytest.raises(ValueError):
        es.run_exhaustive(p, workers=0)


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    p = es.compile_program(M.gen_multiplier_miter(4, "array", "diagonal"))
    with pytest.raises(N.NativeError) as ei:
        es.run_exhaustive(p)
    assert ei.value.code == N.ES_E_NO_DEVICE
