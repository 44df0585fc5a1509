"""AIGER ingest and emission behind the reference's interface.

Mirrors cecprove/aiger.py (parse_aiger :44, write_aiger :197, the error
classes :13-26) and the XOR recovery the CLI applies on load
(transform.detect_xors, transform.py:79-119; cli._load_circuit, cli.py:63-76),
implemented in C++ (csrc/es_aiger.cpp) behind the C ABI (es_aiger_parse,
es_detect_xors, es_aiger_write).  Circuits are built with the reference's
structural hashing, so a parsed file is gate-for-gate the reference's Xag and
compiles to the same ES program.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .xag import Gate, GateKind, Lit, Xag, packed_gates


class AigerError(ValueError):
    pass


class MalformedHeader(AigerError):
    pass


class LatchesUnsupported(AigerError):
    pass


class DanglingLiteral(AigerError):
    pass


_ERRORS = {N.ES_E_AIGER: AigerError, N.ES_E_AIGER_HEADER: MalformedHeader,
           N.ES_E_AIGER_LATCHES: LatchesUnsupported, N.ES_E_AIGER_DANGLING: DanglingLiteral}


def _take(h) -> Xag:
    L = N.lib()
    try:
        n, g, o = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        N.check(L.es_xag_size(h, ctypes.byref(n), ctypes.byref(g), ctypes.byref(o)))
        kind = np.zeros(g.value, np.uint8)
        in0 = np.zeros(g.value, np.uint32)
        in1 = np.zeros(g.value, np.uint32)
        outs = np.zeros(o.value, np.uint32)
        N.check(L.es_xag_read(h, kind.ctypes.data, in0.ctypes.data, in1.ctypes.data, outs.ctypes.data))
    finally:
        L.es_xag_free(h)
    gates = tuple(Gate(GateKind(int(k)), Lit(int(a) >> 1, bool(a & 1)), Lit(int(b) >> 1, bool(b & 1)))
                  for k, a, b in zip(kind, in0, in1))
    return Xag(n.value, gates, tuple(Lit(int(x) >> 1, bool(x & 1)) for x in outs))


def _parse(data, detect: bool) -> Xag:
    if isinstance(data, str):
        data = data.encode()
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    h = ctypes.c_void_p()
    rc = N.lib().es_aiger_parse(buf.ctypes.data if len(buf) else None, len(buf), int(detect),
                                ctypes.byref(h))
    if rc in _ERRORS:
        raise _ERRORS[rc](N.last_error())
    N.check(rc)
    return _take(h)


def parse_aiger(data) -> Xag:
    """Parse ASCII or binary AIGER bytes into an AND-only Xag (aiger.py:44-58)."""
    return _parse(data, False)


def _arrays(xag):
    g = len(xag.gates)
    kind, in0, in1 = packed_gates(xag)
    outs = np.fromiter((o.node * 2 + int(o.neg) for o in xag.outputs), np.uint32, len(xag.outputs))
    return xag.num_pis, g, kind, in0, in1, len(xag.outputs), outs


def detect_xors(xag) -> Xag:
    """Fold the three-AND XOR pattern back into XOR gates (transform.py:79-119)."""
    n, g, kind, in0, in1, no, outs = _arrays(xag)
    h = ctypes.c_void_p()
    N.check(N.lib().es_detect_xors(n, g, kind.ctypes.data, in0.ctypes.data, in1.ctypes.data, no,
                                   outs.ctypes.data, ctypes.byref(h)))
    return _take(h)


def write_aiger(xag) -> bytes:
    """ASCII AIGER bytes; XOR gates become NOT(NOT(a AND NOT b) AND NOT(NOT a AND b))
    (aiger.py:197-225)."""
    n, g, kind, in0, in1, no, outs = _arrays(xag)
    L = N.lib()
    size = N.check(L.es_aiger_write(n, g, kind.ctypes.data, in0.ctypes.data, in1.ctypes.data, no,
                                    outs.ctypes.data, None, 0))
    buf = ctypes.create_string_buffer(size)
    N.check(L.es_aiger_write(n, g, kind.ctypes.data, in0.ctypes.data, in1.ctypes.data, no,
                             outs.ctypes.data, buf, size))
    return buf.raw[:size]


def load_circuit(path: str) -> Xag:
    """The CLI's loader (cli.py:63-76): parse, then recover XORs."""
    with open(path, "rb") as fh:
        return _parse(fh.read(), True)
