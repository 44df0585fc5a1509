"""K4 modules (csrc/k4_skeleton.cu, es_sass.cpp k4_body / k4_module): no GPU.

A K4 module holds many programs' direct-SASS bodies behind the skeleton's
indirect branch (BRXU through the jump table in constant bank 2).  Here a
module is disassembled with cuobjdump (NVIDIA's decoder checks every
encoding, the dispatch prologue included), each body is located through the
jump table, interpreted from its entry to its branch to the RET over numpy
words, and compared with the CPU model of the mapped program (es.map_eval)
-- first failing cofactor copy and its number, as the skeleton folds them.
The branch-target attribute the driver sees must list the rebased BRXU and
the bodies' entries."""
import ctypes
import re
import struct
import subprocess

import numpy as np
import pytest

from paper_2512_06627_b200 import _native as N
from paper_2512_06627_b200 import es
from paper_2512_06627_b200 import miter as M
from paper_2512_06627_b200 import sass_template as S
from tests.test_sass import CUOBJDUMP, M32, expand, interpret


def k4_cubin(progs, ks, variant=0):
    L = N.lib()
    n = len(progs)
    arr = (N.EsProg * n)(*[p.as_struct() for p in progs])
    kk = (ctypes.c_int32 * n)(*ks)
    st = (ctypes.c_int32 * (4 * n + 4))()
    size = N.check(L.es_k4_cubin(arr, n, kk, variant, st, None, 0))
    buf = ctypes.create_string_buffer(size)
    N.check(L.es_k4_cubin(arr, n, kk, variant, st, buf, size))
    regs = dict(zip(("lo", "hi", "o0", "o1"), list(st)[4 * n:]))
    return buf.raw[:size], [st[4 * i] for i in range(n)], regs


def sections(cubin):
    return {name: (off, size) for name, _, off, size in S._sections(cubin)}


@pytest.mark.parametrize("variant", [0, 1])
def test_module_bodies_match_cpu_model(tmp_path, variant):
    xs = [M.flip_gate(M.gen_multiplier_miter(8, "array", "booth"), 300),
          M.gen_multiplier_miter(8, "array", "wallace"),
          M.gen_adder_miter(10),
          M.flip_gate(M.gen_multiplier_miter(10, "array", "booth"), 250)]
    ks = [3, 0, 2, 4]
    if variant == 1:  # the 2-CTA template's ~90 registers: the multiplier miters need more
        xs, ks = xs[1:3], ks[1:3]
    progs = [es.compile_program(x) for x in xs]
    cubin, instrs, regs = k4_cubin(progs, ks, variant)
    sec = sections(cubin)
    toff, _ = sec[".nv.constant2.es_k4"]
    table = struct.unpack_from(f"<{len(progs)}I", cubin, toff)
    path = tmp_path / "k4.cubin"
    path.write_bytes(cubin)
    out = subprocess.run([CUOBJDUMP, "-sass", str(path)], capture_output=True, text=True, check=True).stdout
    ins = [(int(a, 16), t.strip()) for a, t in re.findall(r"/\*([0-9a-f]{4,6})\*/\s+([^;]*);", out)]
    at = {a: i for i, (a, _) in enumerate(ins)}
    # the dispatch: one BRXU, and the attribute lists it and the entries
    brx = [(a, t) for a, t in ins if t.startswith("BRX")]
    assert len(brx) == 1 and brx[0][1].startswith("BRXU")
    ioff, isz = S._nv_info_attr(cubin, ".nv.info.es_k4", S.EIATTR_INDIRECT_BRANCH_TARGETS)
    boff, _, cnt = struct.unpack_from("<III", cubin, ioff)
    assert boff == brx[0][0] and cnt == S.K4_TARGETS
    assert struct.unpack_from(f"<{len(progs)}I", cubin, ioff + 12) == table
    rng = np.random.default_rng(1)
    for i, (p, k) in enumerate(zip(progs, ks)):
        body = []
        for a, t in ins[at[table[i]]:]:
            if t.startswith("BRA"):
                assert ins[at[int(t.split()[-1], 16)]][1].startswith("RET.REL")
                break
            body.append(t)
        assert len(body) == instrs[i]
        ms = es.map_stats(p, k)
        cof = ms["cofactor_pis"]
        kbits = max(p.num_pis - 5 - len(cof), 0)
        wk = rng.integers(0, 1 << kbits, size=24, dtype=np.uint64) if kbits else np.zeros(24, np.uint64)
        R = interpret(body, {regs["lo"]: wk & M32, regs["hi"]: wk >> np.uint64(32)})
        fw_want, fc_want = [], []
        for w in wk:
            fw = fc = 0
            for c in range(1 << len(cof)):
                v = int(es.map_eval(p, expand(w, cof, c), 1, k)[0])
                if v:
                    fw, fc = v, c
                    break
            fw_want.append(fw)
            fc_want.append(fc)
        fw_want = np.array(fw_want, np.uint64)
        np.testing.assert_array_equal(R[regs["o0"]], fw_want, err_msg=f"body {i}")
        hit = fw_want != 0
        np.testing.assert_array_equal(R[regs["o1"]][hit], np.array(fc_want, np.uint64)[hit])
        if variant == 0 and i in (0, 3):
            assert hit.any()


def test_too_wide_body_needs_the_1cta_variant():
    p = es.compile_program(M.flip_gate(M.gen_multiplier_miter(12, "array", "booth"), 250))
    with pytest.raises(N.NativeError):
        k4_cubin([p], [4], 1)
    k4_cubin([p], [4], 0)
